"""FEMNIST CNN clients on the B200 (BASELINE.json config 2).

The reference only ships the multinomial logistic model; config 2 names the
LEAF FEMNIST CNN.  This module is its host side:

* ``CnnLayout`` -- the engine's padded parameter layout (csrc/cnn.cu) and the
  conversion to / from torch's canonical tensors (conv [out,in,5,5], fc
  [out,in], fc1 input flattened (c, h, w));
* ``init_cnn_params`` -- torch-default-style uniform init from a PCG64 seed;
* ``CnnFederation`` -- DeviceFederation whose ``train`` runs the CNN engine
  (``fedhc_cnn_local_train``: conv2 / fc1 / fc2 forward, data and weight
  gradients of every client as grouped tcgen05 GEMMs -- conv2 as implicit
  GEMMs over 4-D TMA boxes -- conv1 (1 input channel, K = 25) fused with
  pooling on the CUDA cores, one CUDA graph per round) and whose ``correct`` runs
  ``fedhc_cnn_eval``.  Plans, permutations, descriptors and FedAvg are the
  linear path's (the round structure of engine.run_experiment does not depend
  on the model).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _abi
from .experiment import DeviceFederation, delta_buffer
from .training import stream_ptr

CANONICAL = ["conv1.weight", "conv1.bias", "conv2.weight", "conv2.bias", "fc1.weight", "fc1.bias", "fc2.weight",
             "fc2.bias"]


class CnnLayout:
    """Padded parameter vector of the engine <-> canonical tensors."""

    def __init__(self, n_classes: int):
        if not 2 <= n_classes <= 64:
            raise ValueError("the CNN engine supports 2..64 classes")
        self.n_classes = n_classes
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_cnn_param_count(C.byref(n)))
        self.P = n.value
        offs = (C.c_int64 * 8)()
        _abi.check(_abi.lib.fedhc_cnn_param_offsets(offs))
        self.off = dict(zip(CANONICAL, list(offs)))

    @property
    def canonical_count(self) -> int:
        c = self.n_classes
        return 32 * 25 + 32 + 64 * 800 + 64 + 2048 * 3136 + 2048 + c * 2048 + c

    def to_padded(self, p: dict[str, np.ndarray]) -> np.ndarray:
        c, o = self.n_classes, self.off
        v = np.zeros(self.P, dtype=np.float64)
        w1 = np.zeros((64, 32))
        w1[:25] = np.asarray(p["conv1.weight"]).reshape(32, 25).T
        v[o["conv1.weight"]:o["conv1.weight"] + 64 * 32] = w1.ravel()
        v[o["conv1.bias"]:o["conv1.bias"] + 32] = p["conv1.bias"]
        # [pair = kh*3 + kw//2][kw % 2][ci][co]; kw = 5 and pair 15 are zero padding (csrc/cnn.cu)
        w2 = np.zeros((5, 6, 32, 64))
        w2[:, :5] = np.asarray(p["conv2.weight"]).transpose(2, 3, 1, 0)
        v[o["conv2.weight"]:o["conv2.weight"] + 15 * 64 * 64] = w2.ravel()
        v[o["conv2.bias"]:o["conv2.bias"] + 64] = p["conv2.bias"]
        f1 = np.zeros((2048, 3200))
        f1[:, :3136] = np.asarray(p["fc1.weight"]).reshape(2048, 64, 7, 7).transpose(0, 2, 3, 1).reshape(2048, 3136)
        v[o["fc1.weight"]:o["fc1.weight"] + 2048 * 3200] = f1.ravel()
        v[o["fc1.bias"]:o["fc1.bias"] + 2048] = p["fc1.bias"]
        f2 = np.zeros((64, 2048))
        f2[:c] = p["fc2.weight"]
        v[o["fc2.weight"]:o["fc2.weight"] + 64 * 2048] = f2.ravel()
        v[o["fc2.bias"]:o["fc2.bias"] + c] = p["fc2.bias"]
        return v

    def from_padded(self, v) -> dict[str, np.ndarray]:
        v = np.asarray(v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
        c, o = self.n_classes, self.off
        w1 = v[o["conv1.weight"]:o["conv1.weight"] + 64 * 32].reshape(64, 32)
        w2 = v[o["conv2.weight"]:o["conv2.weight"] + 15 * 64 * 64].reshape(5, 6, 32, 64)[:, :5]
        f1 = v[o["fc1.weight"]:o["fc1.weight"] + 2048 * 3200].reshape(2048, 3200)
        f2 = v[o["fc2.weight"]:o["fc2.weight"] + 64 * 2048].reshape(64, 2048)
        return {
            "conv1.weight": w1[:25].T.reshape(32, 1, 5, 5).copy(),
            "conv1.bias": v[o["conv1.bias"]:o["conv1.bias"] + 32].copy(),
            "conv2.weight": w2.transpose(3, 2, 0, 1).copy(),
            "conv2.bias": v[o["conv2.bias"]:o["conv2.bias"] + 64].copy(),
            "fc1.weight": f1[:, :3136].reshape(2048, 7, 7, 64).transpose(0, 3, 1, 2).reshape(2048, 3136).copy(),
            "fc1.bias": v[o["fc1.bias"]:o["fc1.bias"] + 2048].copy(),
            "fc2.weight": f2[:c].copy(),
            "fc2.bias": v[o["fc2.bias"]:o["fc2.bias"] + c].copy(),
        }

    def padding_mask(self) -> np.ndarray:
        """True at entries that are layout padding (must stay exactly zero)."""
        return self.to_padded({k: np.ones_like(v) for k, v in init_cnn_params(self.n_classes, 0).items()}) == 0


def init_cnn_params(n_classes: int, seed: int) -> dict[str, np.ndarray]:
    """Uniform(-1/sqrt(fan_in), 1/sqrt(fan_in)) per tensor, fp64, PCG64(seed), canonical order."""
    rng = np.random.default_rng(seed)
    shapes = [((32, 1, 5, 5), 25), ((32,), 25), ((64, 32, 5, 5), 800), ((64,), 800), ((2048, 3136), 3136),
              ((2048,), 3136), ((n_classes, 2048), 2048), ((n_classes,), 2048)]
    out = {}
    for name, (shape, fan_in) in zip(CANONICAL, shapes):
        b = 1.0 / math.sqrt(fan_in)
        out[name] = rng.uniform(-b, b, size=shape)
    return out


class CnnEngine:
    """Owns one fedhc_cnn workspace (activations for max_clients x batch)."""

    def __init__(self, max_clients: int, batch: int, n_classes: int):
        h = C.c_void_p()
        _abi.check(_abi.lib.fedhc_cnn_create(max_clients, batch, n_classes, C.byref(h)))
        self._h = h
        self.max_clients, self.batch, self.n_classes = max_clients, batch, n_classes

    def __del__(self):
        if getattr(self, "_h", None) and getattr(_abi, "lib", None) is not None:
            _abi.lib.fedhc_cnn_destroy(self._h)
        self._h = None

    def local_train(self, desc_ptr: int, k: int, params: torch.Tensor, max_steps: int, lr: float,
                    use_graph: bool = True, stream: int | None = None) -> None:
        s = stream_ptr() if stream is None else stream
        _abi.check(_abi.lib.fedhc_cnn_local_train(self._h, desc_ptr, k, params.data_ptr(), max_steps, float(lr),
                                                  int(use_graph), s))

    def last_loss(self, k: int) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.float32, device="cuda")
        _abi.check(_abi.lib.fedhc_cnn_last_loss(self._h, out.data_ptr(), k, stream_ptr()))
        return out

    def correct_into(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> None:
        """out (dev int64 [1]) += correctly classified rows; no host synchronisation of the result."""
        _abi.check(_abi.lib.fedhc_cnn_eval(self._h, params.data_ptr(), x.data_ptr(), y.data_ptr(), int(y.shape[0]),
                                           out.data_ptr(), stream_ptr()))

    def correct(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> int:
        cnt = torch.zeros(1, dtype=torch.int64, device=params.device)
        self.correct_into(params, x, y, cnt)
        return int(cnt.item())

    KERNELS_PER_STEP = 15     # 9 grouped GEMMs (3 implicit-GEMM conv2) + conv1 fwd/bwd, pool2 fwd/bwd, CE, bias SGD

    def launches_per_round(self, steps: int) -> int:
        """Kernels one fedhc_cnn_local_train launches (broadcast, steps, delta)."""
        return self.KERNELS_PER_STEP * steps + 2


class CnnFederation(DeviceFederation):
    """DeviceFederation with the FEMNIST CNN as the client model (28x28x1 inputs)."""

    def attach_engine(self, max_clients: int, batch: int) -> "CnnFederation":
        if self.n_features != 784:
            raise ValueError("the FEMNIST CNN takes 784-feature (28x28x1) rows")
        self.layout = CnnLayout(self.n_classes)
        self.P = self.layout.P
        self.engine = CnnEngine(max_clients, batch, self.n_classes)
        return self

    def train(self, params: torch.Tensor, participants: list[str], workloads, lr: float, seeds,
              deltas: torch.Tensor | None = None, use_graph: bool = True) -> torch.Tensor:
        k = len(participants)
        if deltas is None:
            deltas = delta_buffer(k, self.P, self.x.device)
        if k == 0:
            return deltas
        meta, perm_bytes = self.stage_plan(participants, workloads, seeds)
        d_desc = self.descriptors(participants, meta, lr, deltas)
        self.last_h2d_bytes = perm_bytes + d_desc.numel()
        max_steps = max(m[2] for m in meta)
        if max(wl.batch_size for wl in workloads) > self.engine.batch:
            raise ValueError("batch size exceeds the CNN workspace")
        self.engine.local_train(d_desc.data_ptr(), k, params, max_steps, lr, use_graph)
        self._keepalive = d_desc
        return deltas

    def correct(self, params: torch.Tensor) -> int:
        if self.n_test == 0:
            return 0
        return self.engine.correct(params, self.x_test, self.y_test)

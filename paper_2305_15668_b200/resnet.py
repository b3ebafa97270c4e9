"""CIFAR ResNet-18 clients on the B200 (BASELINE.json config 3, builder-defined).

Host side of the ResNet engine (csrc/resnet.cu): the padded parameter layout and its conversion to /
from torch's canonical state tensors (conv [out, in, k, k] <-> [k*k*in][out], BN weight / bias /
running_mean / running_var, linear), a torch-default-style initialisation from a PCG64 seed, and
``ResnetFederation`` -- a DeviceFederation whose ``train`` runs fedhc_resnet_local_train (every
convolution of every client as a grouped implicit tcgen05 GEMM, one CUDA graph per round) on
CIFAR-shaped rows (NHWC fp32 [32][32][3] = 3072 features) and whose ``correct`` runs fedhc_resnet_eval
(batch norm with running statistics).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _abi
from .experiment import DeviceFederation, delta_buffer
from .training import stream_ptr

BLOCKS = [(64, 64, 1), (64, 64, 1), (64, 128, 2), (128, 128, 1), (128, 256, 2), (256, 256, 1), (256, 512, 2),
          (512, 512, 1)]
LAYERS = ["layer1.0", "layer1.1", "layer2.0", "layer2.1", "layer3.0", "layer3.1", "layer4.0", "layer4.1"]


def canonical_shapes(n_classes: int) -> list[tuple[str, tuple[int, ...]]]:
    """torch state_dict order (num_batches_tracked excluded) of the CIFAR ResNet-18."""
    out = [("conv1.weight", (64, 3, 3, 3))]

    def bn(prefix, c):
        return [(f"{prefix}.{n}", (c,)) for n in ("weight", "bias", "running_mean", "running_var")]

    out += bn("bn1", 64)
    for name, (ci, co, s) in zip(LAYERS, BLOCKS):
        out.append((f"{name}.conv1.weight", (co, ci, 3, 3)))
        out += bn(f"{name}.bn1", co)
        out.append((f"{name}.conv2.weight", (co, co, 3, 3)))
        out += bn(f"{name}.bn2", co)
        if s != 1 or ci != co:
            out.append((f"{name}.shortcut.0.weight", (co, ci, 1, 1)))
            out += bn(f"{name}.shortcut.1", co)
    out += [("linear.weight", (n_classes, 512)), ("linear.bias", (n_classes,))]
    return out


class ResnetLayout:
    """Padded parameter vector of the engine <-> canonical state tensors."""

    def __init__(self, n_classes: int):
        if not 2 <= n_classes <= 64:
            raise ValueError("the ResNet engine supports 2..64 classes")
        self.n_classes = n_classes
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_resnet_param_count(n_classes, C.byref(n)))
        self.P = n.value
        self.shapes = canonical_shapes(n_classes)
        offs = (C.c_int64 * 128)()
        cnt = C.c_int()
        _abi.check(_abi.lib.fedhc_resnet_param_offsets(n_classes, offs, 128, C.byref(cnt)))
        if cnt.value != len(self.shapes):
            raise RuntimeError("libfedhc ResNet layout does not match the host architecture table")
        self.off = {name: int(offs[i]) for i, (name, _) in enumerate(self.shapes)}

    @property
    def canonical_count(self) -> int:
        return sum(math.prod(s) for _, s in self.shapes)

    @staticmethod
    def _conv_to_engine(w: np.ndarray) -> np.ndarray:
        co, ci, k, _ = w.shape
        return w.transpose(2, 3, 1, 0).reshape(k * k * ci, co)

    def to_padded(self, p: dict[str, np.ndarray]) -> np.ndarray:
        v = np.zeros(self.P, dtype=np.float64)
        for name, shape in self.shapes:
            o = self.off[name]
            a = np.asarray(p[name], dtype=np.float64).reshape(shape)
            flat = self._conv_to_engine(a).ravel() if len(shape) == 4 else a.ravel()
            v[o:o + flat.size] = flat
        return v

    def from_padded(self, v) -> dict[str, np.ndarray]:
        v = np.asarray(v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
        out = {}
        for name, shape in self.shapes:
            o, n = self.off[name], math.prod(shape)
            if len(shape) == 4:
                co, ci, k, _ = shape
                out[name] = v[o:o + n].reshape(k, k, ci, co).transpose(3, 2, 0, 1).copy()
            else:
                out[name] = v[o:o + n].reshape(shape).copy()
        return out

    def padding_mask(self) -> np.ndarray:
        """True at entries that are layout padding (must stay exactly zero)."""
        return self.to_padded({n: np.ones(s) for n, s in self.shapes}) == 0


def init_resnet_params(n_classes: int, seed: int) -> dict[str, np.ndarray]:
    """torch-default init from PCG64(seed): conv / linear U(+-1/sqrt(fan_in)), BN (1, 0, 0, 1)."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape in canonical_shapes(n_classes):
        leaf = name.rsplit(".", 1)[1]
        if len(shape) == 4 or name == "linear.weight" or name == "linear.bias":
            fan_in = 512 if name.startswith("linear") else int(np.prod(shape[1:]))
            b = 1.0 / math.sqrt(fan_in)
            out[name] = rng.uniform(-b, b, size=shape)
        elif leaf in ("weight", "running_var"):
            out[name] = np.ones(shape)
        else:
            out[name] = np.zeros(shape)
    return out


class ResnetEngine:
    """Owns one fedhc_resnet workspace (activations of max_clients x batch images)."""

    KERNELS_PER_STEP = 130   # approximate launch count of one training step (CUDA-graph nodes)

    def __init__(self, max_clients: int, batch: int, n_classes: int):
        h = C.c_void_p()
        _abi.check(_abi.lib.fedhc_resnet_create(max_clients, batch, n_classes, C.byref(h)))
        self._h = h
        self.max_clients, self.batch, self.n_classes = max_clients, batch, n_classes

    def __del__(self):
        if getattr(self, "_h", None) and getattr(_abi, "lib", None) is not None:
            _abi.lib.fedhc_resnet_destroy(self._h)
        self._h = None

    def local_train(self, desc_ptr: int, k: int, params: torch.Tensor, max_steps: int, lr: float,
                    use_graph: bool = True, stream: int | None = None) -> None:
        s = stream_ptr() if stream is None else stream
        _abi.check(_abi.lib.fedhc_resnet_local_train(self._h, desc_ptr, k, params.data_ptr(), max_steps, float(lr),
                                                     int(use_graph), s))

    def last_loss(self, k: int) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.float32, device="cuda")
        _abi.check(_abi.lib.fedhc_resnet_last_loss(self._h, out.data_ptr(), k, stream_ptr()))
        return out

    def launch_count(self) -> int:
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_resnet_launch_count(self._h, C.byref(n)))
        return n.value

    def correct_into(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> None:
        _abi.check(_abi.lib.fedhc_resnet_eval(self._h, params.data_ptr(), x.data_ptr(), y.data_ptr(),
                                              int(y.shape[0]), out.data_ptr(), stream_ptr()))

    def correct(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> int:
        cnt = torch.zeros(1, dtype=torch.int64, device=params.device)
        self.correct_into(params, x, y, cnt)
        return int(cnt.item())


class ResnetFederation(DeviceFederation):
    """DeviceFederation with CIFAR ResNet-18 clients (rows = NHWC fp32 32x32x3)."""

    def attach_engine(self, max_clients: int, batch: int) -> "ResnetFederation":
        if self.n_features != 3072:
            raise ValueError("ResNet-18 clients take 3072-feature (32x32x3 NHWC) rows")
        self.layout = ResnetLayout(self.n_classes)
        self.P = self.layout.P
        self.engine = ResnetEngine(max_clients, batch, self.n_classes)
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
        if max(wl.batch_size for wl in workloads) > self.engine.batch:
            raise ValueError("batch size exceeds the ResNet workspace")
        self.engine.local_train(d_desc.data_ptr(), k, params, max(m[2] for m in meta), lr, use_graph)
        self._keepalive = d_desc
        return deltas

    def correct(self, params: torch.Tensor) -> int:
        if self.n_test == 0:
            return 0
        return self.engine.correct(params, self.x_test, self.y_test)

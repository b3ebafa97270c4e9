"""CIFAR MobileNetV2 clients on the B200 (BASELINE.json config 4, builder-defined).

Host side of the MobileNetV2 engine (csrc/mobilenet.cu): the architecture table, the padded
parameter layout (every channel count rounded up to a multiple of 64; the padding entries are zero and stay
zero) and its conversion to / from torch's canonical state tensors, a torch-default-style initialisation
from a PCG64 seed, and ``MobilenetFederation`` -- a DeviceFederation whose ``train`` runs
fedhc_mobilenet_local_train (pointwise convolutions as grouped implicit tcgen05 GEMMs, depthwise 3x3 on
CUDA cores, one CUDA graph per round) on CIFAR-shaped rows (NHWC fp32 [32][32][3] = 3072 features).
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _abi
from .experiment import DeviceFederation, delta_buffer
from .training import stream_ptr

# (expansion, out channels, repeats, first stride) -- the common CIFAR MobileNetV2 table
CFG = [(1, 16, 1, 1), (6, 24, 2, 1), (6, 32, 3, 2), (6, 64, 4, 2), (6, 96, 3, 1), (6, 160, 3, 2), (6, 320, 1, 1)]
HEAD = 1280


def blocks() -> list[tuple[int, int, int, int]]:
    """(cin, planes, cout, stride) of the 17 inverted-residual blocks."""
    out, cin = [], 32
    for e, c, n, s in CFG:
        for i in range(n):
            out.append((cin, e * cin, c, s if i == 0 else 1))
            cin = c
    return out


def pad64(c: int) -> int:
    return (c + 63) // 64 * 64


def canonical_shapes(n_classes: int) -> list[tuple[str, tuple[int, ...], tuple[int, int] | None]]:
    """torch state_dict order (num_batches_tracked excluded): (name, shape, padded engine matrix or None)."""
    out = [("conv1.weight", (32, 3, 3, 3), (64, 64))]

    def bn(prefix, c):
        return [(f"{prefix}.{n}", (c,), None) for n in ("weight", "bias", "running_mean", "running_var")]

    out += bn("bn1", 32)
    for i, (ci, pl, co, s) in enumerate(blocks()):
        p = f"layers.{i}"
        out.append((f"{p}.conv1.weight", (pl, ci, 1, 1), (pad64(ci), pad64(pl))))
        out += bn(f"{p}.bn1", pl)
        out.append((f"{p}.conv2.weight", (pl, 1, 3, 3), (9, pad64(pl))))
        out += bn(f"{p}.bn2", pl)
        out.append((f"{p}.conv3.weight", (co, pl, 1, 1), (pad64(pl), pad64(co))))
        out += bn(f"{p}.bn3", co)
        if s == 1 and ci != co:
            out.append((f"{p}.shortcut.0.weight", (co, ci, 1, 1), (pad64(ci), pad64(co))))
            out += bn(f"{p}.shortcut.1", co)
    out.append(("conv2.weight", (HEAD, 320, 1, 1), (320, HEAD)))
    out += bn("bn2", HEAD)
    out += [("linear.weight", (n_classes, HEAD), None), ("linear.bias", (n_classes,), None)]
    return out


def _conv_to_matrix(w: np.ndarray) -> np.ndarray:
    """[out, in, k, k] -> [(kh, kw, in)][out]; depthwise [C, 1, 3, 3] -> [9][C]."""
    co, ci, k, _ = w.shape
    return w.transpose(2, 3, 1, 0).reshape(k * k * ci, co)


class MobilenetLayout:
    """Padded parameter vector of the engine <-> canonical state tensors."""

    def __init__(self, n_classes: int):
        if not 2 <= n_classes <= 64:
            raise ValueError("the MobileNetV2 engine supports 2..64 classes")
        self.n_classes = n_classes
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_mobilenet_param_count(n_classes, C.byref(n)))
        self.P = n.value
        self.shapes = canonical_shapes(n_classes)
        offs = (C.c_int64 * 512)()
        cnt = C.c_int()
        _abi.check(_abi.lib.fedhc_mobilenet_param_offsets(n_classes, offs, 512, C.byref(cnt)))
        if cnt.value != len(self.shapes):
            raise RuntimeError("libfedhc MobileNetV2 layout does not match the host architecture table")
        self.off = {name: int(offs[i]) for i, (name, _, _) in enumerate(self.shapes)}

    @property
    def canonical_count(self) -> int:
        return sum(math.prod(s) for _, s, _ in self.shapes)

    def to_padded(self, p: dict[str, np.ndarray]) -> np.ndarray:
        v = np.zeros(self.P, dtype=np.float64)
        for name, shape, mat in self.shapes:
            o = self.off[name]
            a = np.asarray(p[name], dtype=np.float64).reshape(shape)
            if mat is None:
                v[o:o + a.size] = a.ravel()
            else:
                m = _conv_to_matrix(a)
                view = v[o:o + mat[0] * mat[1]].reshape(mat)
                view[:m.shape[0], :m.shape[1]] = m
        return v

    def from_padded(self, v) -> dict[str, np.ndarray]:
        v = np.asarray(v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
        out = {}
        for name, shape, mat in self.shapes:
            o = self.off[name]
            if mat is None:
                out[name] = v[o:o + math.prod(shape)].reshape(shape).copy()
            else:
                co, ci, k, _ = shape
                m = v[o:o + mat[0] * mat[1]].reshape(mat)[:k * k * ci, :co]
                out[name] = m.reshape(k, k, ci, co).transpose(3, 2, 0, 1).copy()
        return out

    def padding_mask(self) -> np.ndarray:
        """True at entries that are layout padding (must stay exactly zero)."""
        return self.to_padded({n: np.ones(s) for n, s, _ in self.shapes}) == 0


def init_mobilenet_params(n_classes: int, seed: int) -> dict[str, np.ndarray]:
    """torch-default init from PCG64(seed): conv / linear U(+-1/sqrt(fan_in)), BN (1, 0, 0, 1)."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape, _ in canonical_shapes(n_classes):
        leaf = name.rsplit(".", 1)[1]
        if len(shape) == 4 or name.startswith("linear"):
            fan_in = HEAD if name.startswith("linear") else int(np.prod(shape[1:]))
            b = 1.0 / math.sqrt(fan_in)
            out[name] = rng.uniform(-b, b, size=shape)
        elif leaf in ("weight", "running_var"):
            out[name] = np.ones(shape)
        else:
            out[name] = np.zeros(shape)
    return out


class MobilenetEngine:
    """Owns one fedhc_mobilenet workspace (activations of max_clients x batch images)."""

    def __init__(self, max_clients: int, batch: int, n_classes: int):
        h = C.c_void_p()
        _abi.check(_abi.lib.fedhc_mobilenet_create(max_clients, batch, n_classes, C.byref(h)))
        self._h = h
        self.max_clients, self.batch, self.n_classes = max_clients, batch, n_classes

    def __del__(self):
        if getattr(self, "_h", None) and getattr(_abi, "lib", None) is not None:
            _abi.lib.fedhc_mobilenet_destroy(self._h)
        self._h = None

    def local_train(self, desc_ptr: int, k: int, params: torch.Tensor, max_steps: int, lr: float,
                    use_graph: bool = True, stream: int | None = None, steps=None) -> None:
        """steps: optional per-client step counts, non-increasing (clients in descending-step order); step s
        then runs only the clients that still have work (heterogeneous sample counts, config 4)."""
        s = stream_ptr() if stream is None else stream
        sp = None
        if steps is not None:
            self._steps = np.ascontiguousarray(steps, dtype=np.int32)
            sp = self._steps.ctypes.data
        _abi.check(_abi.lib.fedhc_mobilenet_local_train(self._h, desc_ptr, k, sp, params.data_ptr(), max_steps,
                                                        float(lr), int(use_graph), s))

    def last_loss(self, k: int) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.float32, device="cuda")
        _abi.check(_abi.lib.fedhc_mobilenet_last_loss(self._h, out.data_ptr(), k, stream_ptr()))
        return out

    def launch_count(self) -> int:
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_mobilenet_launch_count(self._h, C.byref(n)))
        return n.value

    def correct_into(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> None:
        _abi.check(_abi.lib.fedhc_mobilenet_eval(self._h, params.data_ptr(), x.data_ptr(), y.data_ptr(),
                                                 int(y.shape[0]), out.data_ptr(), stream_ptr()))

    def correct(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor) -> int:
        cnt = torch.zeros(1, dtype=torch.int64, device=params.device)
        self.correct_into(params, x, y, cnt)
        return int(cnt.item())


class MobilenetFederation(DeviceFederation):
    """DeviceFederation with CIFAR MobileNetV2 clients (rows = NHWC fp32 32x32x3)."""

    def attach_engine(self, max_clients: int, batch: int) -> "MobilenetFederation":
        if self.n_features != 3072:
            raise ValueError("MobileNetV2 clients take 3072-feature (32x32x3 NHWC) rows")
        self.layout = MobilenetLayout(self.n_classes)
        self.P = self.layout.P
        self.engine = MobilenetEngine(max_clients, batch, self.n_classes)
        return self

    def train(self, params: torch.Tensor, participants: list[str], workloads, lr: float, seeds,
              deltas: torch.Tensor | None = None, use_graph: bool = True) -> torch.Tensor:
        k = len(participants)
        if deltas is None:
            deltas = delta_buffer(k, self.P, self.x.device)
        if k == 0:
            return deltas
        meta, perm_bytes = self.stage_plan(participants, workloads, seeds)
        # descending local-step order (stable): later steps run only the clients that still have batches;
        # delta row i stays participant i's
        order = sorted(range(k), key=lambda i: -meta[i][2])
        d_desc = self.descriptors([participants[i] for i in order], [meta[i] for i in order], lr, deltas,
                                  rows=order)
        self.last_h2d_bytes = perm_bytes + d_desc.numel()
        if max(wl.batch_size for wl in workloads) > self.engine.batch:
            raise ValueError("batch size exceeds the MobileNetV2 workspace")
        steps = [meta[i][2] for i in order]
        self.engine.local_train(d_desc.data_ptr(), k, params, steps[0], lr, use_graph, steps=steps)
        self._keepalive = d_desc
        return deltas

    def correct(self, params: torch.Tensor) -> int:
        if self.n_test == 0:
            return 0
        return self.engine.correct(params, self.x_test, self.y_test)

"""CIFAR ShuffleNetV2 x1.0 clients on the B200 (BASELINE.json config 4's other model; builder-defined).

Host side of the ShuffleNetV2 engine (csrc/shufflenet.cu): the architecture table, the padded
parameter layout and its conversion to / from torch's canonical state tensors, a torch-default-style
initialisation from a PCG64 seed, and ``ShufflenetFederation`` (same contract as MobilenetFederation:
per-client step counts, descending-step order, delta rows kept in participant order).

Layout: a stage's activations are stored in "split form" -- the 2h channels of a block output (torch
order, i.e. after the 2-group channel shuffle) as [X1 | X2], each half padded from h to Ph (multiple of 64).
Weights that read such a tensor (the next stage's down-sampling block, the head) map torch input channel
c to row c (c < h) or Ph + c - h; everything else is padded at the end.  Padding entries are zero.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _abi
from .experiment import DeviceFederation, delta_buffer
from .mobilenet import MobilenetEngine
from .training import stream_ptr

STAGES = [(24, 116, 3, 32), (116, 232, 7, 16), (232, 464, 3, 8)]  # (cin, cout, basic blocks, H_in)
HEAD = 1024


def pad64(c: int) -> int:
    return (c + 63) // 64 * 64


def _split_map(h: int) -> np.ndarray:
    """torch channel -> engine channel of a split-form tensor with halves of h (padded to pad64(h))."""
    c = np.arange(2 * h)
    return np.where(c < h, c, pad64(h) + c - h)


def canonical_shapes(n_classes: int):
    """torch state_dict order: (name, shape, engine (rows, cols) or vector length, row map, col map)."""
    out = []

    def bn(prefix, c, size, idx):
        return [(f"{prefix}.{n}", (c,), size, idx, None) for n in ("weight", "bias", "running_mean", "running_var")]

    ident = lambda n: np.arange(n)  # noqa: E731
    out.append(("conv1.weight", (24, 3, 3, 3), (64, 64), ident(27), ident(24)))
    out += bn("bn1", 24, 64, ident(24))
    for s, (cin, cout, nb, _) in enumerate(STAGES):
        mid = cout // 2
        pm = pad64(mid)
        if s == 0:
            pin, imap = 64, ident(cin)
        else:
            hp = cin // 2
            pin, imap = 2 * pad64(hp), _split_map(hp)
        p = f"layer{s + 1}.0"
        out.append((f"{p}.conv1.weight", (cin, 1, 3, 3), (9, pin), ident(9), imap))
        out += bn(f"{p}.bn1", cin, pin, imap)
        out.append((f"{p}.conv2.weight", (mid, cin, 1, 1), (pin, pm), imap, ident(mid)))
        out += bn(f"{p}.bn2", mid, pm, ident(mid))
        out.append((f"{p}.conv3.weight", (mid, cin, 1, 1), (pin, pm), imap, ident(mid)))
        out += bn(f"{p}.bn3", mid, pm, ident(mid))
        out.append((f"{p}.conv4.weight", (mid, 1, 3, 3), (9, pm), ident(9), ident(mid)))
        out += bn(f"{p}.bn4", mid, pm, ident(mid))
        out.append((f"{p}.conv5.weight", (mid, mid, 1, 1), (pm, pm), ident(mid), ident(mid)))
        out += bn(f"{p}.bn5", mid, pm, ident(mid))
        for j in range(1, nb + 1):
            p = f"layer{s + 1}.{j}"
            out.append((f"{p}.conv1.weight", (mid, mid, 1, 1), (pm, pm), ident(mid), ident(mid)))
            out += bn(f"{p}.bn1", mid, pm, ident(mid))
            out.append((f"{p}.conv2.weight", (mid, 1, 3, 3), (9, pm), ident(9), ident(mid)))
            out += bn(f"{p}.bn2", mid, pm, ident(mid))
            out.append((f"{p}.conv3.weight", (mid, mid, 1, 1), (pm, pm), ident(mid), ident(mid)))
            out += bn(f"{p}.bn3", mid, pm, ident(mid))
    out.append(("conv2.weight", (HEAD, 464, 1, 1), (512, HEAD), _split_map(232), ident(HEAD)))
    out += bn("bn2", HEAD, HEAD, ident(HEAD))
    out.append(("linear.weight", (n_classes, HEAD), None, None, None))
    out.append(("linear.bias", (n_classes,), None, None, None))
    return out


def _to_matrix(w: np.ndarray) -> np.ndarray:
    """[out, in, k, k] -> [(kh, kw, in)][out]; depthwise [C, 1, 3, 3] -> [9][C]."""
    co, ci, k, _ = w.shape
    return w.transpose(2, 3, 1, 0).reshape(k * k * ci, co)


class ShufflenetLayout:
    """Padded parameter vector of the engine <-> canonical state tensors."""

    def __init__(self, n_classes: int):
        if not 2 <= n_classes <= 64:
            raise ValueError("the ShuffleNetV2 engine supports 2..64 classes")
        self.n_classes = n_classes
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_shufflenet_param_count(n_classes, C.byref(n)))
        self.P = n.value
        self.shapes = canonical_shapes(n_classes)
        offs = (C.c_int64 * 512)()
        cnt = C.c_int()
        _abi.check(_abi.lib.fedhc_shufflenet_param_offsets(n_classes, offs, 512, C.byref(cnt)))
        if cnt.value != len(self.shapes):
            raise RuntimeError("libfedhc ShuffleNetV2 layout does not match the host architecture table")
        self.off = {spec[0]: int(offs[i]) for i, spec in enumerate(self.shapes)}

    @property
    def canonical_count(self) -> int:
        return sum(math.prod(s[1]) for s in self.shapes)

    def to_padded(self, p: dict[str, np.ndarray]) -> np.ndarray:
        v = np.zeros(self.P, dtype=np.float64)
        for name, shape, eng, rmap, cmap in self.shapes:
            o = self.off[name]
            a = np.asarray(p[name], dtype=np.float64).reshape(shape)
            if eng is None:
                v[o:o + a.size] = a.ravel()
            elif isinstance(eng, int):
                v[o + rmap] = a
            else:
                m = _to_matrix(a)
                view = v[o:o + eng[0] * eng[1]].reshape(eng)
                view[np.ix_(rmap, cmap)] = m
        return v

    def from_padded(self, v) -> dict[str, np.ndarray]:
        v = np.asarray(v.detach().cpu().numpy() if isinstance(v, torch.Tensor) else v, dtype=np.float64)
        out = {}
        for name, shape, eng, rmap, cmap in self.shapes:
            o = self.off[name]
            if eng is None:
                out[name] = v[o:o + math.prod(shape)].reshape(shape).copy()
            elif isinstance(eng, int):
                out[name] = v[o + rmap].copy()
            else:
                co, ci, k, _ = shape
                m = v[o:o + eng[0] * eng[1]].reshape(eng)[np.ix_(rmap, cmap)]
                out[name] = m.reshape(k, k, ci, co).transpose(3, 2, 0, 1).copy()
        return out

    def padding_mask(self) -> np.ndarray:
        return self.to_padded({s[0]: np.ones(s[1]) for s in self.shapes}) == 0


def init_shufflenet_params(n_classes: int, seed: int) -> dict[str, np.ndarray]:
    """torch-default init from PCG64(seed): conv / linear U(+-1/sqrt(fan_in)), BN (1, 0, 0, 1)."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, shape, *_ in canonical_shapes(n_classes):
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


class ShufflenetEngine(MobilenetEngine):
    """Owns one fedhc_shufflenet workspace (same call surface as MobilenetEngine)."""

    _PREFIX = "fedhc_shufflenet"

    def __init__(self, max_clients: int, batch: int, n_classes: int):
        h = C.c_void_p()
        _abi.check(_abi.lib.fedhc_shufflenet_create(max_clients, batch, n_classes, C.byref(h)))
        self._h = h
        self.max_clients, self.batch, self.n_classes = max_clients, batch, n_classes

    def __del__(self):
        if getattr(self, "_h", None) and getattr(_abi, "lib", None) is not None:
            _abi.lib.fedhc_shufflenet_destroy(self._h)
        self._h = None

    def local_train(self, desc_ptr: int, k: int, params: torch.Tensor, max_steps: int, lr: float,
                    use_graph: bool = True, stream: int | None = None, steps=None) -> None:
        s = stream_ptr() if stream is None else stream
        sp = None
        if steps is not None:
            self._steps = np.ascontiguousarray(steps, dtype=np.int32)
            sp = self._steps.ctypes.data
        _abi.check(_abi.lib.fedhc_shufflenet_local_train(self._h, desc_ptr, k, sp, params.data_ptr(), max_steps,
                                                         float(lr), int(use_graph), s))

    def last_loss(self, k: int) -> torch.Tensor:
        out = torch.empty(k, dtype=torch.float32, device="cuda")
        _abi.check(_abi.lib.fedhc_shufflenet_last_loss(self._h, out.data_ptr(), k, stream_ptr()))
        return out

    def launch_count(self) -> int:
        n = C.c_int64()
        _abi.check(_abi.lib.fedhc_shufflenet_launch_count(self._h, C.byref(n)))
        return n.value

    def correct_into(self, params: torch.Tensor, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> None:
        _abi.check(_abi.lib.fedhc_shufflenet_eval(self._h, params.data_ptr(), x.data_ptr(), y.data_ptr(),
                                                  int(y.shape[0]), out.data_ptr(), stream_ptr()))


class ShufflenetFederation(DeviceFederation):
    """DeviceFederation with CIFAR ShuffleNetV2 clients (rows = NHWC fp32 32x32x3)."""

    def attach_engine(self, max_clients: int, batch: int) -> "ShufflenetFederation":
        if self.n_features != 3072:
            raise ValueError("ShuffleNetV2 clients take 3072-feature (32x32x3 NHWC) rows")
        self.layout = ShufflenetLayout(self.n_classes)
        self.P = self.layout.P
        self.engine = ShufflenetEngine(max_clients, batch, self.n_classes)
        return self

    def train(self, params: torch.Tensor, participants: list[str], workloads, lr: float, seeds,
              deltas: torch.Tensor | None = None, use_graph: bool = True) -> torch.Tensor:
        k = len(participants)
        if deltas is None:
            deltas = delta_buffer(k, self.P, self.x.device)
        if k == 0:
            return deltas
        meta, perm_bytes = self.stage_plan(participants, workloads, seeds)
        order = sorted(range(k), key=lambda i: -meta[i][2])
        d_desc = self.descriptors([participants[i] for i in order], [meta[i] for i in order], lr, deltas,
                                  rows=order)
        self.last_h2d_bytes = perm_bytes + d_desc.numel()
        if max(wl.batch_size for wl in workloads) > self.engine.batch:
            raise ValueError("batch size exceeds the ShuffleNetV2 workspace")
        steps = [meta[i][2] for i in order]
        self.engine.local_train(d_desc.data_ptr(), k, params, steps[0], lr, use_graph, steps=steps)
        self._keepalive = d_desc
        return deltas

    def correct(self, params: torch.Tensor) -> int:
        if self.n_test == 0:
            return 0
        return self.engine.correct(params, self.x_test, self.y_test)

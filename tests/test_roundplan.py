"""Native round planning (csrc/roundplan.cpp) against the Python it replaces: CPython's random.sample on the
selector's MT19937 state (engine.py:302, :327), CPython 3.12's float sum, and the round's staging block
(seeds, batch-order metadata, local_train descriptors, FedAvg coefficients). CPU only."""

import ctypes as C
import random

import numpy as np
import pytest

from paper_2305_15668_b200 import _abi
from paper_2305_15668_b200.experiment import CLIENT_DTYPE
from paper_2305_15668_b200.training import n_permutations, stable_seed


@pytest.mark.parametrize("seed", ["1:selection", "7:selection", "abc", 12345])
@pytest.mark.parametrize("n,k", [(128, 100), (10, 10), (1000, 100), (2000, 1000), (40, 5), (40, 6), (7, 0),
                                 (3000, 17), (1, 1), (60, 59)])
def test_native_sample_matches_cpython(seed, n, k):
    py = random.Random(seed)
    st = np.array(py.getstate()[1], dtype=np.uint32)
    out = np.zeros(max(k, 1), np.int32)
    for _ in range(3):  # consecutive rounds: the state carries over
        want = py.sample(range(n), k)
        _abi.check(_abi.lib.fedhc_mt_sample(st.ctypes.data, n, k, out.ctypes.data))
        assert out[:k].tolist() == want
    assert tuple(st.tolist()) == py.getstate()[1]


def test_native_sample_rejects_oversized():
    st = np.array(random.Random(1).getstate()[1], dtype=np.uint32)
    out = np.zeros(4, np.int32)
    with pytest.raises(ValueError, match="Sample larger than population"):
        _abi.check(_abi.lib.fedhc_mt_sample(st.ctypes.data, 3, 4, out.ctypes.data))


def test_py_float_sum_matches_builtin():
    rng = np.random.default_rng(0)
    for x in (rng.integers(16, 1025, 100).astype(np.float64), rng.standard_normal(1000) * 1e10,
              np.array([1e16, 1.0, -1e16, 3.0]), np.zeros(0), np.array([0.1] * 10)):
        x = np.ascontiguousarray(x)
        assert _abi.lib.fedhc_py_float_sum(x.ctypes.data, len(x)) == sum(x.tolist())


def test_round_pack_matches_python_plan():
    rng = np.random.default_rng(3)
    n_fleet, k = 50, 17
    ids = [f"c{i:04d}" for i in range(n_fleet)]
    reprs = [C.c_char_p(repr(c).encode()) for c in ids]
    rptr = np.array([C.cast(b, C.c_void_p).value for b in reprs], np.uint64)
    ns = rng.integers(16, 700, n_fleet)
    bs = rng.choice([32, 50, 64], n_fleet)
    rows = rng.integers(0, 400, n_fleet)
    steps = -(-ns // bs)
    nperm = np.array([n_permutations(int(r), int(n), int(b)) for r, n, b in zip(rows, ns, bs)], np.int64)
    xptr = rng.integers(1 << 32, 1 << 40, n_fleet).astype(np.uint64)
    yptr = rng.integers(1 << 32, 1 << 40, n_fleet).astype(np.uint64)
    w = ns.astype(np.float64)
    mine = rng.choice(n_fleet, k, replace=False).astype(np.int64)
    total = float(sum(w[mine].tolist()) + 123.0)
    perm_base, delta_base, stride, lr, seed, r = 0x7f0000000000, 0x7e0000000000, 31408, 0.1, 3, 5
    buf = np.zeros(k * (24 + CLIENT_DTYPE.itemsize + 8), np.uint8)
    words, mr = C.c_int64(), C.c_int32()
    r32, p32, s32, b32 = (a.astype(np.int32) for a in (rows, nperm, steps, bs))  # keep the buffers alive
    _abi.check(_abi.lib.fedhc_round_pack(seed, r, k, mine.ctypes.data, rptr.ctypes.data,
                                         r32.ctypes.data, p32.ctypes.data, s32.ctypes.data, b32.ctypes.data,
                                         xptr.ctypes.data, yptr.ctypes.data, w.ctypes.data, total, lr, perm_base,
                                         delta_base, stride, buf.ctypes.data, C.byref(words), C.byref(mr)))
    sizes = rows[mine] * nperm[mine]
    offs = np.concatenate([[0], np.cumsum(sizes)[:-1]]).astype(np.int64)
    assert words.value == int(sizes.sum()) and mr.value == int(rows[mine].max())
    rng_seeds = [stable_seed("local_train", stable_seed("train", seed, r, ids[c])) for c in mine]
    assert buf[:8 * k].view(np.uint64).tolist() == rng_seeds
    assert buf[8 * k:12 * k].view(np.int32).tolist() == rows[mine].tolist()
    assert buf[12 * k:16 * k].view(np.int32).tolist() == nperm[mine].tolist()
    assert buf[16 * k:24 * k].view(np.int64).tolist() == offs.tolist()
    d = buf[24 * k:24 * k + k * CLIENT_DTYPE.itemsize].view(CLIENT_DTYPE)
    assert d["x"].tolist() == xptr[mine].tolist() and d["y"].tolist() == yptr[mine].tolist()
    assert d["perm"].tolist() == (perm_base + offs * 4).tolist()
    assert d["n_rows"].tolist() == rows[mine].tolist() and d["n_batches"].tolist() == steps[mine].tolist()
    assert d["batch_size"].tolist() == bs[mine].tolist() and np.all(d["lr"] == np.float32(lr))
    assert d["delta"].tolist() == [delta_base + i * stride for i in range(k)]
    coef = buf[24 * k + k * CLIENT_DTYPE.itemsize:].view(np.float64)
    assert coef.tolist() == (w[mine] / total).tolist()

"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/fedhc.h declares, and its host-only entry points (FedAvg
coefficients, cost model) agree with the reference semantics."""

import ctypes as C
import os
import random
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "fedhc.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fedhc_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2305_15668_b200 import _abi
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(_abi.lib, name), name
    assert set(names) <= set(_abi.SIGNATURES), set(names) - set(_abi.SIGNATURES)


def test_library_is_in_tree_and_sm100a():
    from paper_2305_15668_b200 import _abi
    assert os.path.dirname(_abi.LIB_PATH) == os.path.join(ROOT, "paper_2305_15668_b200")
    blob = open(_abi.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_version():
    from paper_2305_15668_b200 import _abi
    assert _abi.lib.fedhc_version() == 1


def _coef(weights):
    from paper_2305_15668_b200 import _abi
    n = len(weights)
    arr = (C.c_double * max(n, 1))(*weights)
    out = (C.c_double * max(n, 1))()
    st = _abi.lib.fedhc_fedavg_coefficients(arr, n, out)
    return st, list(out)[:n], _abi.lib.fedhc_last_error().decode()


def test_fedavg_coefficients_match_python_sum():
    rng = random.Random(7)
    for _ in range(500):
        n = rng.randint(1, 40)
        w = [rng.choice([rng.uniform(0, 1e6), rng.uniform(0, 1e-3), float(rng.randint(1, 1024)), 1e16, 1.0])
             for _ in range(n)]
        st, coef, _ = _coef(w)
        assert st == 0
        total = float(sum(w))
        assert coef == [x / total for x in w]


def test_fedavg_coefficient_errors():
    from paper_2305_15668_b200 import _abi
    assert _coef([]) [0] == _abi.ERR_AGGREGATION
    st, _, msg = _coef([1.0, -1.0])
    assert st == _abi.ERR_AGGREGATION and msg == "weights must be non-negative"
    st, _, msg = _coef([0.0, 0.0])
    assert st == _abi.ERR_AGGREGATION and msg == "weights must not all be zero"


def test_status_maps_to_reference_exceptions():
    from paper_2305_15668_b200 import _abi
    from paper_2305_15668_b200.errors import AggregationError, ConfigError
    _coef([-1.0])
    with pytest.raises(AggregationError, match="non-negative"):
        _abi.check(_abi.ERR_AGGREGATION)
    with pytest.raises(ConfigError):
        _abi.check(_abi.ERR_CONFIG)


def test_kernels_present_in_sass():
    """The CUDA kernels are compiled for sm_100a and use the tensor pipe (HMMA) + TMA bulk copies."""
    import shutil
    import subprocess
    from paper_2305_15668_b200 import _abi
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "-sass", _abi.LIB_PATH], capture_output=True, text=True).stdout
    for kernel in ("train_c64_kernel", "train_tc_kernel", "train_generic_kernel", "train_pipe_kernel", "train_fused_kernel",
                   "train_pipe2_kernel", "fedavg_kernel", "eval_kernel",
                   "grouped_gemm_kernel", "conv1_fwd_kernel", "conv1_bwd_kernel", "perm_kernel"):
        assert kernel in out, kernel
    assert "HMMA" in out and "UBLKCP" in out
    # tcgen05 grouped GEMM: UMMA issue, TMA tensor loads and the TMA-store epilogue
    assert "UTCHMMA" in out and "UTMALDG" in out and "UTMASTG" in out

"""ctypes binding of libfedhc.so (include/fedhc.h).

The library is built in-tree by ``paper_2305_15668_b200/build.py`` (called
from ``__graft_entry__.build()``).  There is deliberately no fallback: if the
library is missing, importing the compute API raises ``ImportError``.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import AggregationError, ConfigError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfedhc.so")

OK, ERR_VALUE, ERR_AGGREGATION, ERR_CONFIG, ERR_CUDA, ERR_UNSUPPORTED, ERR_RUNTIME = range(7)
F32, F64 = 0, 1

EV_LAUNCHED, EV_PHASE, EV_TRAINED, EV_UPLOADED, EV_SLOT_FREED, EV_ROUND_COMPLETE, EV_ALLOC, EV_INSTRUCTION = range(8)


class FedhcCudaError(RuntimeError):
    """A CUDA runtime failure inside libfedhc."""


class Client(C.Structure):
    _fields_ = [
        ("x", C.c_void_p),
        ("y", C.c_void_p),
        ("perm", C.c_void_p),
        ("n_rows", C.c_int32),
        ("n_batches", C.c_int32),
        ("batch_size", C.c_int32),
        ("lr", C.c_float),
        ("delta", C.c_void_p),
    ]


class DesClient(C.Structure):
    _fields_ = [
        ("budget", C.c_int32),
        ("num_samples", C.c_int32),
        ("batch_size", C.c_int32),
        ("model_layers", C.c_int32),
        ("seq_len", C.c_int32),
        ("extra_model_factor", C.c_double),
        ("n_phases", C.c_int32),
        ("phase_frac", C.POINTER(C.c_double)),
        ("phase_demand", C.POINTER(C.c_double)),
    ]


class DesConfig(C.Structure):
    _fields_ = [
        ("theta", C.c_double),
        ("max_executors", C.c_int32),
        ("scheduler", C.c_int32),
        ("dynamic_parallelism", C.c_int32),
        ("alpha", C.c_double),
        ("beta", C.c_double),
        ("launch_latency", C.c_double),
        ("terminate_latency", C.c_double),
        ("upload_latency", C.c_double),
    ]


class DesEvent(C.Structure):
    _fields_ = [
        ("t", C.c_double),
        ("kind", C.c_int32),
        ("client", C.c_int32),
        ("executor", C.c_int32),
        ("aux", C.c_int32),
        ("budget", C.c_double),
        ("alloc_off", C.c_int64),
        ("alloc_len", C.c_int32),
        ("pad_", C.c_int32),
    ]


class DesReport(C.Structure):
    _fields_ = [
        ("makespan", C.c_double),
        ("utilization", C.c_double),
        ("vacancy_area", C.c_double),
        ("throughput", C.c_double),
        ("degenerate", C.c_int32),
        ("n_events", C.c_int32),
        ("n_alloc_pairs", C.c_int64),
    ]


class RunnerConfig(C.Structure):
    """fedhc_runner_config (include/fedhc.h)."""
    _fields_ = [
        ("reprs", C.c_void_p), ("rows", C.c_void_p), ("n_perms", C.c_void_p), ("n_batches", C.c_void_p),
        ("batch_size", C.c_void_p), ("xptr", C.c_void_p), ("yptr", C.c_void_p), ("weight", C.c_void_p),
        ("over_theta", C.c_void_p), ("sim_index", C.c_void_p), ("mt_state", C.c_void_p), ("sim", C.c_void_p),
        ("des_clients", C.c_void_p), ("des_ids", C.c_void_p),
        ("params", C.c_void_p), ("deltas", C.c_void_p), ("delta_stride_bytes", C.c_int64),
        ("split_offset", C.c_int64), ("x_test", C.c_void_p), ("y_test", C.c_void_p), ("n_test", C.c_int64),
        ("correct_dev", C.c_void_p), ("correct_host", C.c_void_p), ("stage_host", C.c_void_p),
        ("stage_dev", C.c_void_p), ("plan_dev", C.c_void_p), ("plan_cap_words", C.c_int64),
        ("plan_stream", C.c_void_p), ("eval_stream", C.c_void_p), ("seed", C.c_int64),
        ("async_host", C.c_void_p), ("async_dev", C.c_void_p), ("snapshots", C.c_void_p),
        ("des_cfg", DesConfig), ("lr", C.c_float),
        ("n_fleet", C.c_int32), ("participants", C.c_int32), ("slots", C.c_int32), ("n_features", C.c_int32),
        ("n_classes", C.c_int32), ("max_batch", C.c_int32), ("split", C.c_int32), ("eval_ctas", C.c_int32),
        ("rows_max", C.c_int32), ("async_buffer", C.c_int32),
    ]


class RunnerPlanInfo(C.Structure):
    """fedhc_runner_plan_info (include/fedhc.h)."""
    _fields_ = [
        ("selected", C.c_void_p), ("starts", C.c_void_p), ("ends", C.c_void_p), ("launch_order", C.c_void_p),
        ("upload_order", C.c_void_p), ("par_t", C.c_void_p), ("par_n", C.c_void_p), ("chunk_end", C.c_void_p),
        ("par_cap", C.c_int32),
        ("n_launched", C.c_int32), ("n_uploaded", C.c_int32), ("n_par", C.c_int32), ("over_theta", C.c_int32),
        ("degenerate", C.c_int32), ("max_rows", C.c_int32), ("n_chunks", C.c_int32),
        ("makespan", C.c_double), ("utilization", C.c_double), ("vacancy_area", C.c_double),
        ("throughput", C.c_double), ("total_weight", C.c_double), ("perm_words", C.c_int64),
        ("h2d_bytes", C.c_int64),
    ]


class GemmArgs(C.Structure):
    _fields_ = [
        ("G", C.c_int32), ("M", C.c_int32), ("N", C.c_int32), ("K", C.c_int32),
        ("a_mn", C.c_int32), ("b_mn", C.c_int32),
        ("A", C.c_void_p), ("B", C.c_void_p),
        ("epilogue", C.c_int32), ("bias_per_row", C.c_int32),
        ("D", C.c_void_p), ("ldd", C.c_int64), ("d_gstride", C.c_int64),
        ("bias", C.c_void_p), ("bias_gstride", C.c_int64),
        ("master", C.c_void_p), ("shadow", C.c_void_p), ("lr", C.c_float), ("pad_", C.c_int32),
        ("mask", C.c_void_p), ("rowsum", C.c_void_p), ("a_gstride", C.c_int64), ("b_gstride", C.c_int64),
        ("lda", C.c_int64), ("ldb", C.c_int64),
    ]


EPI_F32, EPI_BF16, EPI_BIAS_RELU_BF16, EPI_SGD, EPI_RELU_MASK_BF16 = range(5)

_vp, _i, _i64, _d, _dp = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.POINTER(C.c_double)

SIGNATURES = {
    "fedhc_last_error": (C.c_char_p, []),
    "fedhc_version": (_i, []),
    "fedhc_device_info": (_i, [_i, C.POINTER(_i), C.POINTER(_i), C.POINTER(_i)]),
    "fedhc_local_train": (_i, [_vp, _i, _vp, _i, _i, _i, _vp]),
    "fedhc_x_split": (_i, [_vp, _i64, _i, _vp, _vp]),
    "fedhc_pcg64_standard_normal": (_i, [_vp, _i64, _vp, _vp, _vp]),
    "fedhc_runner_create": (_i, [_vp, _vp]),
    "fedhc_runner_destroy": (None, [_vp]),
    "fedhc_runner_plan": (_i, [_vp, _i64, _d, _i, _vp]),
    "fedhc_runner_launch": (_i, [_vp, _i, _vp]),
    "fedhc_runner_result": (_i, [_vp, _i, _vp]),
    "fedhc_local_train_split": (_i, [_vp, _i, _vp, _i, _i, _i, _i64, _vp]),
    "fedhc_tc_trace_read": (_i, [_vp]),
    "fedhc_mt_sample": (_i, [_vp, _i, _i, _vp]),
    "fedhc_py_float_sum": (C.c_double, [_vp, _i]),
    "fedhc_round_pack": (_i, [C.c_int64, C.c_int64, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, C.c_double,
                              C.c_float, C.c_uint64, C.c_uint64, C.c_int64, _vp, _vp, _vp]),
    "fedhc_loss_and_grad": (_i, [_vp, _vp, _i, _i, _i, _vp, _vp, _vp, _vp, _vp]),
    "fedhc_fedavg_coefficients": (_i, [_dp, _i, _dp]),
    "fedhc_fedavg": (_i, [_vp, _vp, _i64, _i, _vp, _i, _vp, _vp, _i64, _vp]),
    "fedhc_eval": (_i, [_vp, _vp, _i64, _i, _i, _vp, _vp, _vp]),
    "fedhc_eval_ctas": (_i, [_vp, _vp, _i64, _i, _i, _vp, _vp, _i, _vp]),
    "fedhc_des_create": (_vp, []),
    "fedhc_des_destroy": (None, [_vp]),
    "fedhc_des_run_round": (
        _i,
        [_vp, C.POINTER(DesClient), C.POINTER(C.c_char_p), C.POINTER(C.c_int32), _i, C.POINTER(DesConfig), _d, _i,
         _i, _dp, _dp, C.POINTER(DesReport)],
    ),
    "fedhc_des_trace": (
        _i,
        [_vp, C.POINTER(C.POINTER(DesEvent)), C.POINTER(C.POINTER(C.c_int32)), C.POINTER(_dp), C.POINTER(_dp),
         C.POINTER(C.POINTER(C.c_int32)), C.POINTER(_i)],
    ),
    "fedhc_work_units": (_d, [_i, _i, _i, _i, _d, _d, _d]),
    "fedhc_batch_permutations": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i]),
    "fedhc_batch_permutations_device": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _vp]),
    "fedhc_pcg64_state": (_i, [C.c_uint64, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                C.POINTER(C.c_uint64)]),
    "fedhc_maxmin_allocate": (_i, [_dp, _dp, _i, _d, _dp]),
    "fedhc_round_seeds": (_i, [_i64, _i64, C.POINTER(C.c_char_p), _i, _vp, _vp]),
    "fedhc_sha256_le32": (C.c_uint32, [C.c_char_p, _i64]),
    "fedhc_gctx_pool_create": (_i, [_i, _i, C.POINTER(_vp), C.POINTER(_i), C.POINTER(_i)]),
    "fedhc_gctx_pool_destroy": (None, [_vp]),
    "fedhc_gctx_stream": (_i, [_vp, _i, _i, C.POINTER(_vp), C.POINTER(_i)]),
    "fedhc_gctx_stream_rest": (_i, [_vp, _i, _i, C.POINTER(_vp), C.POINTER(_i)]),
    "fedhc_probe_smid": (_i, [_vp, _i, _vp]),
    "fedhc_gemm_bf16_tn": (_i, [_i, _i, _i, _i, _vp, _vp, _vp, _vp]),
    "fedhc_gemm": (_i, [C.POINTER(GemmArgs), _vp]),
    "fedhc_cnn_param_count": (_i, [C.POINTER(C.c_int64)]),
    "fedhc_cnn_param_offsets": (_i, [C.POINTER(C.c_int64)]),
    "fedhc_cnn_create": (_i, [_i, _i, _i, C.POINTER(C.c_void_p)]),
    "fedhc_cnn_destroy": (_i, [_vp]),
    "fedhc_cnn_local_train": (_i, [_vp, _vp, _i, _vp, _i, C.c_float, _i, _vp]),
    "fedhc_cnn_last_loss": (_i, [_vp, _vp, _i, _vp]),
    "fedhc_cnn_eval": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "fedhc_cnn_conv2": (_i, [_i, _i, _i, _vp, _vp, _vp, _vp, _vp, C.c_float, _vp]),
    "fedhc_nhwc_conv": (_i, [_i] * 9 + [_vp, _vp, _vp, _vp, _vp, C.c_float, _vp]),
    "fedhc_resnet_param_count": (_i, [_i, _vp]),
    "fedhc_resnet_param_offsets": (_i, [_i, _vp, _i, _vp]),
    "fedhc_resnet_create": (_i, [_i, _i, _i, _vp]),
    "fedhc_resnet_destroy": (_i, [_vp]),
    "fedhc_resnet_local_train": (_i, [_vp, _vp, _i, _vp, _i, C.c_float, _i, _vp]),
    "fedhc_resnet_last_loss": (_i, [_vp, _vp, _i, _vp]),
    "fedhc_resnet_launch_count": (_i, [_vp, _vp]),
    "fedhc_resnet_eval": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "fedhc_dw_conv": (_i, [_i, _i, _i, _i, _i, _i, _vp, _vp, _vp, _vp, _vp, C.c_float, _vp]),
    "fedhc_mobilenet_param_count": (_i, [_i, _vp]),
    "fedhc_mobilenet_param_offsets": (_i, [_i, _vp, _i, _vp]),
    "fedhc_mobilenet_create": (_i, [_i, _i, _i, _vp]),
    "fedhc_mobilenet_destroy": (_i, [_vp]),
    "fedhc_mobilenet_local_train": (_i, [_vp, _vp, _i, _vp, _vp, _i, C.c_float, _i, _vp]),
    "fedhc_mobilenet_last_loss": (_i, [_vp, _vp, _i, _vp]),
    "fedhc_mobilenet_launch_count": (_i, [_vp, _vp]),
    "fedhc_mobilenet_eval": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "fedhc_shufflenet_param_count": (_i, [_i, _vp]),
    "fedhc_shufflenet_param_offsets": (_i, [_i, _vp, _i, _vp]),
    "fedhc_shufflenet_create": (_i, [_i, _i, _i, _vp]),
    "fedhc_shufflenet_destroy": (_i, [_vp]),
    "fedhc_shufflenet_local_train": (_i, [_vp, _vp, _i, _vp, _vp, _i, C.c_float, _i, _vp]),
    "fedhc_shufflenet_last_loss": (_i, [_vp, _vp, _i, _vp]),
    "fedhc_shufflenet_launch_count": (_i, [_vp, _vp]),
    "fedhc_shufflenet_eval": (_i, [_vp, _vp, _vp, _vp, _i64, _vp, _vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"libfedhc.so not found at {LIB_PATH}; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(status: int) -> None:
    """Map a libfedhc status to the reference's exception types."""
    if status == OK:
        return
    msg = lib.fedhc_last_error().decode(errors="replace")
    if status == ERR_AGGREGATION:
        raise AggregationError(msg)
    if status == ERR_CONFIG:
        raise ConfigError(msg)
    if status == ERR_VALUE:
        raise ValueError(msg)
    if status == ERR_RUNTIME:
        raise RuntimeError(msg)
    if status == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise FedhcCudaError(msg)

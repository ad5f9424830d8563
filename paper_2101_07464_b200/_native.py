"""ctypes binding of the C-ABI in include/hd.h (libhd_b200.so, built in-tree).

This is the only way the Python layer reaches the device path: there is no
CPU fallback. If the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HD_LIB overrides the library path (A/B measurements of alternative builds)
LIB_PATH = os.environ.get("HD_LIB") or os.path.join(_HERE, "lib", "libhd_b200.so")

HD_OK = 0
HD_ERR_INVALID_ARGUMENT = 1
HD_ERR_BUDGET_EXHAUSTED = 2
HD_ERR_RESOURCE_CAP = 3
HD_ERR_RUNTIME = 4
HD_ERR_CUDA = 5
HD_ERR_NCCL = 6

HD_GINIBRE, HD_HAAR, HD_GOE = 0, 1, 2
HD_RIGHT, HD_LEFT = 0, 1
HD_F64, HD_F32, HD_C128 = 0, 1, 2
HD_DRAWS_PHILOX, HD_DRAWS_INJECTED, HD_DRAWS_REFERENCE = 0, 1, 2
DRAW_MODES = {"philox": HD_DRAWS_PHILOX, "injected": HD_DRAWS_INJECTED, "reference": HD_DRAWS_REFERENCE}
SIGN_RULES = {"stable": 0, "negative_at_zero": 1, "zero_when_negative": 2}
UPDATES = {"identity": 0, "normalize": 1, "tanh_mix": 2}
SIDE_RULES = {"alternate": 0, "right": 1, "left": 2}

# Every symbol include/hd.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "hd_create", "hd_destroy", "hd_shape", "hd_remaining", "hd_counts", "hd_chain_sizes", "hd_probe",
    "hd_push_draws", "hd_reset", "hd_run", "hd_run_callback", "hd_set_profiling", "hd_get_stats",
    "hd_reset_stats", "hd_launch_count", "hd_last_error", "hd_version", "hd_reflector_apply",
    "hd_run_async", "hd_wait", "hd_reseed", "hd_rs_create", "hd_rs_destroy", "hd_rs_next_u64", "hd_rs_uniform",
    "hd_rs_normal", "hd_rs_normal_vector", "hd_rs_bernoulli_gaussian", "hd_derive_seed",
    "hd_philox_normals", "hd_batch_run", "hd_exchange_create_local", "hd_exchange_nccl_id", "hd_exchange_create_nccl", "hd_exchange_destroy",
    "hd_shard_plan", "hd_shard_range", "hd_run_amp", "hd_run_spiked",
)
_NON_STATUS = ("hd_last_error", "hd_version", "hd_rs_destroy", "hd_rs_next_u64", "hd_rs_uniform", "hd_rs_normal",
               "hd_derive_seed")


class hd_config(C.Structure):
    _fields_ = [
        ("ensemble", C.c_int32), ("dtype", C.c_int32), ("m", C.c_int64), ("n", C.c_int64),
        ("sigma", C.c_double), ("seed", C.c_uint64), ("stream", C.c_uint64), ("capacity", C.c_int64),
        ("draw_mode", C.c_int32), ("skip_reflector", C.c_int32), ("sign_rule", C.c_int32),
        ("device", C.c_int32), ("shard_count", C.c_int32), ("shard_rank", C.c_int32), ("exchange", C.c_void_p),
    ]


class hd_run_args(C.Structure):
    _fields_ = [
        ("update", C.c_int32), ("side_rule", C.c_int32), ("iterations", C.c_int64), ("x1", C.c_void_p),
        ("x0", C.c_void_p), ("on_device", C.c_int32), ("use_graph", C.c_int32), ("traj", C.c_void_p),
        ("final_out", C.c_void_p), ("stream", C.c_void_p),
    ]


class hd_amp_args(C.Structure):
    _fields_ = [
        ("beta", C.c_void_p), ("w", C.c_void_p), ("iterations", C.c_int64), ("alpha", C.c_double),
        ("x_out", C.c_void_p), ("mse_out", C.c_void_p), ("on_device", C.c_int32), ("use_graph", C.c_int32),
        ("stream", C.c_void_p),
    ]


class hd_spiked_args(C.Structure):
    _fields_ = [
        ("u", C.c_void_p), ("x1", C.c_void_p), ("iterations", C.c_int64), ("theta", C.c_double),
        ("x_out", C.c_void_p), ("overlap_out", C.c_void_p), ("on_device", C.c_int32), ("use_graph", C.c_int32),
        ("stream", C.c_void_p),
    ]


class hd_batch_item(C.Structure):
    _fields_ = [("x1", C.c_void_p), ("out", C.c_void_p), ("seed", C.c_uint64)]


class hd_kernel_stats(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("launches", C.c_int64), ("ms", C.c_double), ("alg_bytes", C.c_double)]


UPDATE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_void_p,
                        C.c_int64, C.c_void_p)
SIDE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int64)

_lib = None


class BudgetExhausted(RuntimeError):
    """types.hpp:32-35 (registered by module.cpp:42)."""


class ResourceCapExceeded(RuntimeError):
    """types.hpp:39-43 (registered by module.cpp:43)."""


class HDCudaError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libhd_b200.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.hd_last_error.restype = C.c_char_p
        L.hd_version.restype = C.c_char_p
        L.hd_create.argtypes = [C.POINTER(hd_config), C.POINTER(vp)]
        L.hd_destroy.argtypes = [vp]
        L.hd_shape.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.hd_remaining.argtypes = [vp, C.POINTER(i64)]
        L.hd_counts.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.hd_chain_sizes.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        L.hd_probe.argtypes = [vp, vp, i64, vp, i64, i32, i32, vp]
        L.hd_push_draws.argtypes = [vp, vp, i64, i32]
        L.hd_reset.argtypes = [vp]
        L.hd_run.argtypes = [vp, C.POINTER(hd_run_args)]
        L.hd_run_callback.argtypes = [vp, i64, i32, C.POINTER(vp), SIDE_FN, UPDATE_FN, vp, vp]
        L.hd_set_profiling.argtypes = [vp, i32]
        L.hd_get_stats.argtypes = [vp, C.POINTER(hd_kernel_stats), i32, C.POINTER(i32)]
        L.hd_reset_stats.argtypes = [vp]
        L.hd_launch_count.argtypes = [vp, C.POINTER(i64)]
        L.hd_reflector_apply.argtypes = [vp, i64, i64, C.c_double, i32, vp, vp, i64, i32, vp]
        L.hd_run_async.argtypes = [vp, C.POINTER(hd_run_args)]
        L.hd_run_amp.argtypes = [vp, C.POINTER(hd_amp_args)]
        L.hd_run_spiked.argtypes = [vp, C.POINTER(hd_spiked_args)]
        L.hd_wait.argtypes = [vp]
        L.hd_reseed.argtypes = [vp, C.c_uint64]
        L.hd_rs_create.argtypes = [C.c_uint64, C.c_uint64, C.POINTER(vp)]
        L.hd_rs_destroy.argtypes = [vp]
        L.hd_rs_destroy.restype = None
        L.hd_rs_next_u64.argtypes = [vp]
        L.hd_rs_next_u64.restype = C.c_uint64
        L.hd_rs_uniform.argtypes = [vp]
        L.hd_rs_uniform.restype = C.c_double
        L.hd_rs_normal.argtypes = [vp]
        L.hd_rs_normal.restype = C.c_double
        L.hd_rs_normal_vector.argtypes = [vp, i64, vp]
        L.hd_rs_bernoulli_gaussian.argtypes = [vp, i64, C.c_double, C.c_double, vp]
        L.hd_derive_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.hd_philox_normals.argtypes = [C.c_uint64, C.c_uint64, i64, i64, vp, vp]
        L.hd_batch_run.argtypes = [C.POINTER(vp), i32, C.POINTER(hd_run_args), C.POINTER(hd_batch_item)]
        L.hd_exchange_create_local.argtypes = [i32, C.POINTER(vp)]
        L.hd_exchange_nccl_id.argtypes = [vp]
        L.hd_exchange_create_nccl.argtypes = [vp, i32, i32, i32, C.POINTER(vp)]
        L.hd_exchange_destroy.argtypes = [vp]
        L.hd_shard_plan.argtypes = [i64, i32, i32, i64, C.POINTER(i64), C.POINTER(i64)]
        L.hd_shard_range.argtypes = [vp, i32, C.POINTER(i64), C.POINTER(i64)]
        L.hd_derive_seed.restype = C.c_uint64
        for name in EXPORTS:
            if name not in _NON_STATUS:
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == HD_OK:
        return
    msg = lib().hd_last_error().decode()
    if rc == HD_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == HD_ERR_BUDGET_EXHAUSTED:
        raise BudgetExhausted(msg)
    if rc == HD_ERR_RESOURCE_CAP:
        raise ResourceCapExceeded(msg)
    if rc == HD_ERR_CUDA:
        raise HDCudaError(msg)
    raise RuntimeError(msg)

"""ctypes binding of the C ABI in include/hawkes_b200.h.

The shared library is built in-tree (`make`, or __graft_entry__.build()) as
paper_2407_11349_b200/libhawkes_b200.so.  There is no fallback: importing
this module without the library raises ImportError.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

import os

# HK_LIB overrides the library path (tuning experiments with alternative
# kernel shapes, see tools/tune_shapes.sh).
LIB_PATH = Path(os.environ.get("HK_LIB") or Path(__file__).resolve().parent / "libhawkes_b200.so")

if not LIB_PATH.exists():
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `make` (or __graft_entry__.build()); "
        "the B200 engine has no CPU fallback")

lib = C.CDLL(str(LIB_PATH))

HK_OK, HK_INVALID_ARGUMENT, HK_OUT_OF_RANGE, HK_RUNTIME_ERROR, HK_NOT_IMPLEMENTED = range(5)
HK_OPT_BG_EXPANSION = 1
HK_OPT_FGT = 2
HK_OPT_BG_FGT = 3
HK_OPT_TR_CUT = 4
HK_OPT_CELLS = 5
HK_OPT_SINGLE_FP64 = 6


class hk_params(C.Structure):
    _fields_ = [("mu0", C.c_double), ("tau_t", C.c_double), ("xi0", C.c_double),
                ("sigma_x", C.c_double), ("sigma_t", C.c_double), ("area", C.c_double),
                ("variant", C.c_int)]


_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_szp = np.ctypeslib.ndpointer(dtype=np.uintp, flags="C_CONTIGUOUS")
_sz = C.c_size_t
_ctx = C.c_void_p
_pp = C.POINTER(hk_params)

# (name, restype, argtypes) for every symbol declared in include/hawkes_b200.h
SIGNATURES = [
    ("hk_create", C.c_int, [_dp, _dp, _dp, _dp, _sz, C.c_int, C.POINTER(_ctx)]),
    ("hk_create_variant", C.c_int, [_dp, _dp, _dp, _dp, _sz, C.c_int, C.c_int, C.POINTER(_ctx)]),
    ("hk_create_devices", C.c_int, [_dp, _dp, _dp, _dp, _sz, np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"),
                                   C.c_int, C.c_int, C.POINTER(_ctx)]),
    ("hk_create_shard", C.c_int, [_dp, _dp, _dp, _dp, _sz, _sz, _sz, C.c_int, C.POINTER(_ctx)]),
    ("hk_destroy", None, [_ctx]),
    ("hk_set_locations", C.c_int, [_ctx, _dp, _dp]),
    ("hk_set_locations_device", C.c_int, [_ctx, C.c_void_p, C.c_void_p]),
    ("hk_eval", C.c_int, [_ctx, _pp, C.POINTER(C.c_double), C.c_void_p]),
    ("hk_eval_detail", C.c_int, [_ctx, _pp, C.POINTER(C.c_double), C.c_void_p, C.c_void_p, C.c_void_p]),
    ("hk_eval_single", C.c_int, [_ctx, _pp, C.POINTER(C.c_double)]),
    ("hk_ws_eval", C.c_int, [_ctx, _pp, C.c_int, C.POINTER(C.c_double), C.c_void_p]),
    ("hk_ws_eval_single", C.c_int, [_ctx, _pp, C.c_int, C.POINTER(C.c_double)]),
    ("hk_ws_stats", C.c_int, [_ctx, C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    ("hk_eval_async", C.c_int, [_ctx, _pp, C.c_int]),
    ("hk_result_device", C.c_void_p, [_ctx]),
    ("hk_stream", C.c_void_p, [_ctx, C.c_int]),
    ("hk_regions_create", C.c_int, [_sz, np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"), _dp,
                                   _szp, _szp, _szp, _dp, C.c_void_p, _sz,
                                   np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS"), C.c_int,
                                   C.POINTER(C.c_void_p)]),
    ("hk_regions_destroy", None, [C.c_void_p]),
    ("hk_regions_sample", C.c_int, [C.c_void_p, C.c_uint64, C.c_uint64, _dp, _dp]),
    ("hk_resample_locations", C.c_int, [_ctx, C.c_void_p, C.c_uint64, C.c_uint64]),
    ("hk_eval_rows", C.c_int, [_ctx, _pp, _sz, _sz, _dp, C.c_void_p]),
    ("hk_set_option", C.c_int, [_ctx, C.c_int, C.c_int]),
    ("hk_fgt_stats", C.c_int, [_ctx, C.POINTER(C.c_long), C.POINTER(C.c_long), C.POINTER(C.c_int)]),
    ("hk_rows", C.c_int, [_ctx, C.POINTER(_sz), C.POINTER(_sz), C.POINTER(C.c_int)]),
    ("hk_set_profiling", C.c_int, [_ctx, C.c_int]),
    ("hk_profile", C.c_int, [_ctx, C.POINTER(C.c_double), C.POINTER(C.c_long), C.POINTER(C.c_long)]),
    ("hk_reset_profile", C.c_int, [_ctx]),
    ("hk_profile_kinds", C.c_int, [_ctx, _dp, np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")]),
    ("hk_validate_catalog", C.c_int, [_dp, _dp, _dp, _dp, _sz]),
    ("hk_validate_params", C.c_int, [_pp]),
    ("hk_partition_make", C.c_int, [_sz, _sz, _szp]),
    ("hk_plan_shards", C.c_int, [_dp, _sz, _sz, _szp]),
    ("hk_plan_shards_variant", C.c_int, [_dp, _sz, _sz, C.c_int, _szp]),
    ("hk_benchmark_catalog", C.c_int, [_sz, C.c_uint64, _dp, _dp, _dp, _dp]),
    ("hk_measure_fp64_peak", C.c_int, [C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    ("hk_last_error", C.c_char_p, []),
    ("hk_version", C.c_char_p, []),
]

for _name, _res, _args in SIGNATURES:
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


class CudaRuntimeError(RuntimeError):
    """HK_RUNTIME_ERROR: a CUDA runtime failure inside the engine."""


def check(rc: int) -> None:
    """Maps the ABI's return codes onto the Python equivalents of the
    reference's exceptions (invalid_argument -> ValueError, out_of_range ->
    IndexError)."""
    if rc == HK_OK:
        return
    msg = (lib.hk_last_error() or b"").decode()
    if rc == HK_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == HK_OUT_OF_RANGE:
        raise IndexError(msg)
    if rc == HK_NOT_IMPLEMENTED:
        raise NotImplementedError(msg)
    raise CudaRuntimeError(msg)

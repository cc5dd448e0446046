"""ctypes binding of libpfb200.so (the C ABI declared in include/pfb200.h).

This module is the only place that touches the native library.  There is no
fallback: if the shared object is missing the import of the device engine
fails loudly, and every device entry point raises when no CUDA device exists.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_int32, c_int64, c_uint8, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# PFB200_LIB selects an alternative build of the same library (A/B kernel
# experiments in scripts/); the default is the in-tree build.
LIB_PATH = os.environ.get("PFB200_LIB") or os.path.join(_HERE, "_native", "libpfb200.so")

PFB_BLOCK = 4096
PFB_NLIMBS = 68
PFB_ACC_WORDS = 72
PFB_ACC_FAILS = 71
PFB_MAX_DALITZ_TERMS = 16

# status codes (enum pfb_status)
OK = 0
E_NONPOSITIVE_DENSITY = 1
E_NONFINITE_DENSITY = 2
E_NEGATIVE_DENSITY = 3
E_FRACTION_OUT_OF_RANGE = 4
E_EMPTY_DATASET = 5
E_NONPOSITIVE_NORM = 6
E_DEGENERATE_GRID = 7
E_INVALID_SUM = 8
E_NONPOSITIVE_EXPECTATION = 9
E_ENVELOPE_HIT = 10
E_ATTEMPTS_EXHAUSTED = 11
E_PEER_TIMEOUT = 12
E_UNBOUNDED_OBSERVABLE = 13
E_OUT_OF_BOUNDS = 14
E_INVALID_ARGUMENT = 20
E_UNSUPPORTED_PLAN = 21
E_CUDA = 30
E_NO_DEVICE = 31
E_OUT_OF_MEMORY = 32

# node kinds (enum pfb_kind)
KIND_CODES = {
    "gaussian": 1,
    "exponential": 2,
    "polynomial": 3,
    "add": 4,
    "prod": 5,
    "dalitz": 6,
}

EVALUATORS = {0: "literal", 1: "sum-of-products", 2: "dalitz", 3: "dalitz-cached"}


class PfbNode(ctypes.Structure):
    _fields_ = [
        ("kind", c_int32),
        ("nchild", c_int32),
        ("col0", c_int32),
        ("col1", c_int32),
        ("nparam", c_int32),
        ("aux", c_int32),
    ]


class PfbDalitzDesc(ctypes.Structure):
    _fields_ = [
        ("mother_mass", c_double),
        ("m1", c_double),
        ("m2", c_double),
        ("m3", c_double),
        ("nterms", c_int32),
        ("pair", c_int32 * PFB_MAX_DALITZ_TERMS),
        ("spin", c_int32 * PFB_MAX_DALITZ_TERMS),
    ]


NORM_CONST, NORM_GAUSSIAN, NORM_EXPONENTIAL, NORM_DALITZ, NORM_QUADRATURE = 0, 1, 2, 3, 4


class PfbObjNode(ctypes.Structure):
    _fields_ = [("norm_kind", c_int32), ("weight_col", c_int32), ("lo", c_double), ("hi", c_double),
                ("value", c_double), ("quad_plan", c_void_p), ("quad_rule", c_void_p)]


class PfbErr(ctypes.Structure):
    _fields_ = [("code", c_int32), ("node", c_int32), ("index", c_int64), ("value", c_double)]


class PfbPcg64(ctypes.Structure):
    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64), ("inc_hi", ctypes.c_uint64),
                ("inc_lo", ctypes.c_uint64)]


class PfbGenStats(ctypes.Structure):
    _fields_ = [("attempts", c_int64), ("accepted", c_int64), ("in_boundary", c_int64), ("produced", c_int64),
                ("observed", c_double), ("ambiguous", c_int64)]


_PTR = c_void_p
_DBL_P = POINTER(c_double)
_I64_P = POINTER(c_int64)

# (name, restype, argtypes)
_SIGNATURES = [
    ("pfb_version", c_int, []),
    ("pfb_strerror", ctypes.c_char_p, [c_int]),
    ("pfb_device_count", c_int, [POINTER(c_int)]),
    ("pfb_ctx_create", c_int, [c_int, POINTER(_PTR)]),
    ("pfb_ctx_destroy", c_int, [_PTR]),
    ("pfb_ctx_set_stream", c_int, [_PTR, _PTR]),
    ("pfb_ctx_stream", _PTR, [_PTR]),
    ("pfb_ctx_synchronize", c_int, [_PTR]),
    ("pfb_ctx_set_warps_per_block", c_int, [_PTR, c_int]),
    ("pfb_ctx_set_pipeline", c_int, [_PTR, c_int]),
    ("pfb_ctx_launch_count", c_int, [_PTR, _I64_P]),
    ("pfb_ctx_enable_timing", c_int, [_PTR, c_int]),
    ("pfb_ctx_last_kernel_ms", c_int, [_PTR, POINTER(c_float)]),
    ("pfb_store_create", c_int, [_PTR, c_int32, c_int64, POINTER(_PTR)]),
    ("pfb_store_upload", c_int, [_PTR, c_int32, _DBL_P, c_int64, c_int64]),
    ("pfb_store_wrap", c_int, [_PTR, c_int32, c_int64, POINTER(_PTR), POINTER(_PTR)]),
    ("pfb_store_device_ptr", c_int, [_PTR, c_int32, POINTER(_PTR)]),
    ("pfb_store_destroy", c_int, [_PTR]),
    ("pfb_plan_compile", c_int, [_PTR, POINTER(PfbNode), c_int32, POINTER(PfbDalitzDesc), c_int32, POINTER(_PTR)]),
    ("pfb_plan_destroy", c_int, [_PTR]),
    ("pfb_plan_evaluator", c_int, [_PTR, POINTER(c_int32)]),
    ("pfb_plan_set_lineshape_cache", c_int, [_PTR, c_int32]),
    ("pfb_plan_cache_recomputes", c_int, [_PTR, _I64_P]),
    ("pfb_nll", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int64, _DBL_P, c_int32, _DBL_P, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_nll_block_sums", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int64, _DBL_P, c_int32, _DBL_P, c_int32, _DBL_P, c_int64, POINTER(PfbErr)]),
    ("pfb_nll_batch", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int64, _DBL_P, c_int32, c_int32, _DBL_P, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_nll_partial_async", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int64, _DBL_P, c_int32, _DBL_P, c_int32, _PTR]),
    ("pfb_nll_enqueue", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, _DBL_P, c_int32, _DBL_P, c_int32, _PTR, _PTR]),
    ("pfb_finalize", c_int, [_PTR, _PTR, _DBL_P, _I64_P]),
    ("pfb_last_error", c_int, [_PTR, POINTER(PfbErr)]),
    ("pfb_ctx_last_fraction_failure", c_int, [_PTR, POINTER(c_int32)]),
    ("pfb_objective_create", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int32, POINTER(c_int32), _DBL_P,
                                     POINTER(PfbObjNode), _DBL_P, POINTER(_PTR)]),
    ("pfb_objective_eval", c_int, [_PTR, _DBL_P, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_objective_eval_batch", c_int, [_PTR, _DBL_P, c_int32, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_objective_set_matrix", c_int, [_PTR, _DBL_P]),
    ("pfb_objective_set_bounds", c_int, [_PTR, _DBL_P, _DBL_P]),
    ("pfb_objective_destroy", c_int, [_PTR]),
    ("pfb_objective_set_persistent", c_int, [_PTR, c_int32]),
    ("pfb_ctx_persist_stop", c_int, [_PTR]),
    ("pfb_ctx_persist_trace", c_int, [_PTR, POINTER(ctypes.c_uint64)]),
    ("pfb_quadrature", c_int, [_PTR, _PTR, _PTR, c_int32, _DBL_P, c_int32, _DBL_P, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_nll_host", c_int, [_PTR, _PTR, POINTER(_DBL_P), c_int32, c_int64, _DBL_P, c_int32, _DBL_P, c_int32, _DBL_P, POINTER(PfbErr)]),
    ("pfb_terms_block_sums", c_int, [_PTR, _DBL_P, c_int64, _DBL_P, _DBL_P]),
    ("pfb_exact_sum_host", c_int, [_DBL_P, c_int64, _DBL_P]),
    ("pfb_acc_round", c_int, [_I64_P, _DBL_P]),
    ("pfb_acc_add_host", c_int, [_I64_P, _DBL_P, c_int64]),
    ("pfb_shard_bounds", c_int, [c_int64, c_int32, c_int64, _I64_P]),
    ("pfb_grid_create", c_int, [_PTR, POINTER(PfbDalitzDesc), c_int32, c_int32, POINTER(_PTR)]),
    ("pfb_grid_info", c_int, [_PTR, _I64_P, _DBL_P]),
    ("pfb_grid_mask", c_int, [_PTR, POINTER(c_uint8)]),
    ("pfb_grid_integrals", c_int, [_PTR, _PTR, c_int32, POINTER(c_int32), POINTER(c_int32), _DBL_P, POINTER(c_uint8), POINTER(c_uint8), _DBL_P]),
    ("pfb_grid_destroy", c_int, [_PTR]),
    ("pfb_gen_dalitz", c_int, [_PTR, POINTER(PfbDalitzDesc), _DBL_P, c_double, ctypes.c_uint64, c_int64, _PTR, _I64_P]),
    ("pfb_gen_1d", c_int, [_PTR, c_int32, c_double, c_double, c_double, c_double, c_double, c_double, ctypes.c_uint64, c_int64, _PTR]),
    ("pfb_store_download", c_int, [_PTR, c_int32, _DBL_P, c_int64, c_int64]),
    ("pfb_fp64_peak", c_int, [_PTR, _DBL_P]),
    ("pfb_ctx_spin", c_int, [_PTR, c_int64, _PTR, c_int64]),
    ("pfb_peer_create", c_int, [_PTR, c_int32, c_int32, _PTR]),
    ("pfb_peer_open", c_int, [_PTR, _PTR]),
    ("pfb_peer_attach", c_int, [_PTR, _PTR]),
    ("pfb_peer_mailbox", c_int, [_PTR, POINTER(_PTR)]),
    ("pfb_peer_allreduce", c_int, [_PTR, _PTR, c_double]),
    ("pfb_nll_peer", c_int, [_PTR, _PTR, _PTR, c_int64, c_int64, c_int64, _DBL_P, c_int32, _DBL_P, c_int32,
                             c_double, POINTER(c_double), POINTER(c_int32)]),
    ("pfb_read_bw", c_int, [_PTR, _PTR, c_int64, c_int32, c_int32, c_int32, _DBL_P]),
    ("pfb_overhead_probe", c_int, [_PTR, c_int32, c_int32, _DBL_P]),
    ("pfb_npy_length", c_int, [ctypes.c_char_p, _I64_P]),
    ("pfb_store_load_npy", c_int, [_PTR, c_int32, ctypes.c_char_p, c_int64, c_int64, c_int64]),
    ("pfb_store_check_range", c_int, [_PTR, c_int32, c_int64, c_int64, c_double, c_double, _I64_P, _DBL_P]),
    ("pfb_pcg_scan_1d", c_int, [_PTR, _PTR, _DBL_P, c_int32, _DBL_P, c_int32, c_double, c_double, c_int64, _DBL_P]),
    ("pfb_pcg_scan_dalitz", c_int, [_PTR, POINTER(PfbDalitzDesc), _DBL_P, c_int32, _DBL_P]),
    ("pfb_pcg_generate_1d", c_int, [_PTR, _PTR, _DBL_P, c_int32, _DBL_P, c_int32, c_double, c_double, c_double,
                                    POINTER(PfbPcg64), c_int64, c_int64, _PTR, c_int64, POINTER(PfbGenStats)]),
    ("pfb_pcg_generate_dalitz", c_int, [_PTR, POINTER(PfbDalitzDesc), _DBL_P, c_double, POINTER(PfbPcg64), c_int64,
                                        c_int64, _PTR, c_int64, POINTER(PfbGenStats)]),
    ("pfb_bin_fill", c_int, [_PTR, _PTR, c_int64, c_int64, c_int32, _PTR, _PTR, _PTR, _PTR, _PTR]),
    ("pfb_binned_nll", c_int, [_PTR, _PTR, _PTR, _PTR, c_int64, c_double, c_double, _PTR, c_int32, _PTR, c_int32,
                               _DBL_P, _PTR]),
]

EXPORTED = tuple(name for name, _, _ in _SIGNATURES)

_lib = None


class NativeMissing(RuntimeError):
    """libpfb200.so is not built (run __graft_entry__.build() or `make`)."""


def lib():
    """Load libpfb200.so once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeMissing(f"{LIB_PATH} not found: build the CUDA engine first (make)")
    handle = ctypes.CDLL(LIB_PATH)
    for name, restype, argtypes in _SIGNATURES:
        fn = getattr(handle, name)
        fn.restype = restype
        fn.argtypes = argtypes
    _lib = handle
    return _lib


def strerror(code: int) -> str:
    return lib().pfb_strerror(code).decode()


class NativeError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} (status {code})")


def check(code: int, where: str) -> None:
    if code != OK:
        raise NativeError(code, where)


def dptr(arr) -> ctypes.POINTER(c_double):
    """double* to a C-contiguous float64 numpy array."""
    return arr.ctypes.data_as(_DBL_P)


def device_count() -> int:
    n = c_int(0)
    check(lib().pfb_device_count(ctypes.byref(n)), "pfb_device_count")
    return n.value

"""ctypes binding of include/bart_b200.h (the drop-in boundary).

There is no CPU fallback: if `lib/libbart_b200.so` cannot be loaded, or no
CUDA device is visible, every call raises.  Status codes map to the
reference's exceptions: BART_EINVAL -> ValueError (sampler.py:214-217,
trees.py:63-67), anything else -> RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from ._build import LIB

BART_OK, BART_EINVAL, BART_ECUDA, BART_ESTATE, BART_ERANGE = 0, 1, 2, 3, 4
MAX_DEPTH = 8
SHARD_HANDLE_BYTES = 256
PROPOSAL_ROWS = 12


class Dims(C.Structure):
    _fields_ = [("n", C.c_int64), ("p", C.c_int32), ("m", C.c_int32), ("max_depth", C.c_int32), ("_pad", C.c_int32)]


class HParams(C.Structure):
    _fields_ = [
        ("leaf_sd", C.c_double), ("lam", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
        ("leaf_mean", C.c_double), ("nu", C.c_double), ("p_grow", C.c_double),
        ("update_sigma", C.c_int32), ("_pad", C.c_int32), ("depth_prob", C.c_double * MAX_DEPTH),
    ]


class TraceOpts(C.Structure):
    _fields_ = [("n_iter", C.c_int64), ("n_keep", C.c_int64), ("n_test", C.c_int64),
                ("store_train_draws", C.c_int32), ("store_forests", C.c_int32), ("train_ring", C.c_int64)]


TRACE_POINTS = 8


class Randoms(C.Structure):
    _fields_ = [("move_u", C.c_void_p), ("accept_u", C.c_void_p), ("leaf_z", C.c_void_p), ("chi2", C.c_double)]


_P = C.c_void_p
_SIGS = {
    "bart_create": [C.POINTER(Dims), C.POINTER(HParams), _P, _P, _P, C.c_double, C.c_uint64, C.c_int, C.POINTER(C.c_void_p)],
    "bart_create_ex": [C.POINTER(Dims), C.POINTER(HParams), _P, _P, _P, C.c_double, C.c_uint64, C.c_int, C.c_int,
                       C.POINTER(C.c_void_p)],
    "bart_destroy": [_P],
    "bart_create_shard": [C.POINTER(Dims), C.c_int64, C.c_int, C.c_int, C.POINTER(HParams), _P, _P, _P, C.c_double,
                          C.c_uint64, C.c_int, C.POINTER(C.c_void_p)],
    "bart_shard_export": [_P, _P],
    "bart_shard_connect": [_P, _P],
    "bart_set_copy_groups": [_P, C.c_int],
    "bart_trace_begin": [_P, C.POINTER(TraceOpts), _P],
    "bart_trace_keep": [_P],
    "bart_trace_counts": [_P, _P, _P],
    "bart_trace_read": [_P] + [_P] * 12,
    "bart_trace_read_draws": [_P, C.c_int64, C.c_int64, _P, _P],
    "bart_set_iteration": [_P, C.c_int64],
    "bart_profile_forest": [_P, C.c_int, _P],
    "bart_get_step_result": [_P, _P, _P],
    "bart_read_step_result": [_P, C.c_int64, _P, _P],
    "bart_trace_end": [_P],
    "bart_grid_minmax": [_P, C.c_int64, C.c_int32, _P, _P, C.c_int],
    "bart_quantize": [_P, C.c_int64, C.c_int32, _P, _P, _P, C.c_int],
    "bart_grid_uniform_quantize": [_P, C.c_int64, C.c_int32, C.c_int32, _P, _P, _P, C.c_int],
    "bart_set_state": [_P, _P, _P, _P, _P, _P, C.c_double],
    "bart_set_hparams": [_P, C.POINTER(HParams)],
    "bart_set_sigma2": [_P, C.c_double],
    "bart_step": [_P, C.POINTER(Randoms)],
    "bart_propose": [_P, _P],
    "bart_run": [_P, C.c_int64],
    "bart_sync": [_P],
    "bart_get_forest": [_P, _P, _P, _P],
    "bart_get_leaf_index": [_P, _P],
    "bart_get_resid": [_P, _P],
    "bart_get_sigma2": [_P, _P],
    "bart_get_accepted": [_P, _P],
    "bart_get_proposals": [_P, _P, _P],
    "bart_get_randoms": [_P, _P, _P, _P, _P],
    "bart_set_exchange": [_P, C.c_int],
    "bart_philox4x32_10": [_P, _P, _P, C.c_int64, C.c_int],
    "bart_set_taps": [_P, C.c_int],
    "bart_get_taps": [_P, _P, _P],
    "bart_predict_cached": [_P, _P],
    "bart_predict_matrix": [_P, _P, C.c_int64, _P],
    "bart_traverse": [C.POINTER(Dims), _P, _P, _P, _P, C.c_int],
    "bart_evaluate": [C.POINTER(Dims), _P, _P, _P, _P, _P, C.c_int],
    "bart_evaluate_many": [C.POINTER(Dims), C.c_int64, _P, _P, _P, _P, _P, C.c_int],
    "bart_sum_leaf_values": [C.POINTER(Dims), _P, _P, _P, C.c_int],
    "bart_profile": [_P, C.c_int64, _P],
    "bart_sweep_config": [_P, _P],
    "bart_run_timed": [_P, C.c_int64, _P],
    "bart_set_timeline": [_P, C.c_int],
    "bart_get_timeline": [_P, _P],
    "bart_get_trace": [_P, _P],
    "bart_graph_active": [_P],
}
_I64 = {"bart_iteration": [_P], "bart_kernel_launches": [_P]}
_I32 = {"bart_device_sms": [C.c_int]}
_STR = {"bart_last_error": [], "bart_version": []}
EXPORTS = sorted(list(_SIGS) + list(_I64) + list(_I32) + list(_STR))

_lib = None


def load_library(path: str | None = None) -> C.CDLL:
    """Load and type the shared library (no device needed).

    BART_LIB overrides the in-tree path (A/B experiments between builds).
    """
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("BART_LIB") or LIB
    if not os.path.exists(path):
        raise RuntimeError(
            f"CUDA library {path} is missing; build it with `python -m paper_2410_23244_b200._build` "
            "(there is no CPU fallback)")
    lib = C.CDLL(path)
    variant = path != LIB  # an A/B build of an older revision may lack newer entry points
    for name, args in _SIGS.items():
        if variant and not hasattr(lib, name):
            continue
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, args in _I64.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int64
    for name, args in _I32.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name, args in _STR.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_char_p
    _lib = lib
    return lib


def lib() -> C.CDLL:
    return load_library()


def check(rc: int) -> None:
    if rc == BART_OK:
        return
    msg = lib().bart_last_error().decode(errors="replace")
    if rc == BART_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(f"bart_b200 error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def dims(n: int, p: int, m: int, max_depth: int) -> Dims:
    return Dims(int(n), int(p), int(m), int(max_depth), 0)


def hparams(hp, depth_probs: np.ndarray) -> HParams:
    h = HParams()
    h.leaf_sd, h.lam, h.alpha, h.beta = float(hp.leaf_sd), float(hp.lam), float(hp.alpha), float(hp.beta)
    h.leaf_mean, h.nu, h.p_grow = float(hp.leaf_mean), float(hp.nu), float(hp.p_grow)
    h.update_sigma = 1 if hp.update_sigma else 0
    for i in range(MAX_DEPTH):
        h.depth_prob[i] = float(depth_probs[i]) if i < len(depth_probs) else 0.0
    return h

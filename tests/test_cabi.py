"""The C-ABI library loads on a CPU-only host and exports what include/*.h declares."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "bart_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bart_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("bart_create", "bart_step", "bart_run", "bart_destroy", "bart_traverse",
                 "bart_predict_cached", "bart_last_error", "bart_set_state"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2410_23244_b200 import _build, _native
    _build.build()
    lib = _native.load_library()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert sorted(_native.EXPORTS) == declared_symbols()
    assert lib.bart_version().startswith(b"bart_b200")


def test_shape_errors_map_to_valueerror_without_device():
    """Argument validation happens before any CUDA call (sampler.py:214-217 semantics)."""
    import numpy as np

    from paper_2410_23244_b200 import _native as N
    lib = N.load_library()
    import ctypes as C
    h = C.c_void_p()
    X = np.zeros((4, 1), np.uint8)
    y = np.zeros(4, np.float32)
    mc = np.array([300], np.int64)  # > 255 cutpoints is rejected (grid.py:18)
    hp = N.hparams(type("H", (), dict(leaf_sd=1, lam=1, alpha=.95, beta=2, leaf_mean=0, nu=3, p_grow=.5,
                                      update_sigma=True))(), np.zeros(8))
    with pytest.raises(ValueError):
        N.check(lib.bart_create(N.dims(4, 1, 1, 3), hp, N.ptr(X), N.ptr(mc), N.ptr(y), 1.0, 0, 0, C.byref(h)))
    with pytest.raises(ValueError, match="max_depth"):
        N.check(lib.bart_create(N.dims(4, 1, 1, 9), hp, N.ptr(X), N.ptr(mc), N.ptr(y), 1.0, 0, 0, C.byref(h)))
    with pytest.raises(ValueError, match="n_trees"):
        N.check(lib.bart_create(N.dims(4, 1, 0, 3), hp, N.ptr(X), N.ptr(mc), N.ptr(y), 1.0, 0, 0, C.byref(h)))


def test_python_init_state_validates_shapes():
    import numpy as np

    from paper_2410_23244_b200.sampler import Hyperparams, init_state
    hp = Hyperparams(leaf_sd=0.1, lam=0.1, n_trees=2, max_depth=3)
    with pytest.raises(ValueError):
        init_state(np.zeros((5, 2), np.uint8), np.array([3, 3]), np.zeros(4), hp, None)
    with pytest.raises(ValueError):
        init_state(np.zeros((5, 2), np.uint8), np.array([3]), np.zeros(5), hp, None)
    with pytest.raises(ValueError):
        init_state(np.zeros((5, 2), np.uint8), np.array([3, 3]), np.zeros(5),
                   Hyperparams(leaf_sd=0.1, lam=0.1, n_trees=2, max_depth=9), None)

"""Forest, trace and chain-state containers.

BFORGE1 (forest) and BFTRACE1 (trace) are the reference's little-endian
formats (bforge/serialize.py:1-29 documents the layouts, 66-188 the
readers/writers): files written here load in the reference and vice versa.

* ``save_forest`` / ``load_forest``: one forest + its cutpoint grid.
* ``save_trace`` / ``load_trace``: a fit() trace.  The JSON header's
  ``config`` holds the reference's FitConfig fields only, so the reference's
  loader accepts the file; this package's extra fields ride in a separate
  ``b200`` header key, which the reference ignores.
* ``TraceFile``: a BFTRACE1 writer that takes the arrays in pieces.  fit()
  uses it to stream the kept training-row draws from the device (one chunk of
  draws at a time) straight into the file, so a trace larger than host
  memory never exists as one host array.
* ``save_checkpoint`` / ``load_checkpoint``: a mid-chain checkpoint (BFCKPT1,
  new: the reference never serializes SamplerState or its RNG) -- forest,
  leaf-index cache, residuals, sigma^2, iteration and the random stream
  (device Philox seed + counter, or the numpy Generator state), from which a
  resumed chain continues bit-identically.
"""

from __future__ import annotations

import dataclasses
import json
import struct
from typing import BinaryIO, Optional

import numpy as np

from .grid import CutpointGrid
from .trees import Forest, heap_size, min_axis_dtype, split_slots

FOREST_MAGIC = b"BFORGE1\0"
TRACE_MAGIC = b"BFTRACE1"
TRACE_VERSION = 1
CHECKPOINT_MAGIC = b"BFCKPT1\0"
CHECKPOINT_VERSION = 1

# bforge.regression.FitConfig's fields, in declaration order (regression.py:34-50)
REFERENCE_CONFIG_FIELDS = ("n_trees", "n_burn", "n_kept", "thinning", "max_depth", "grid", "n_cutpoints", "seed",
                           "k", "q", "nu", "n_chains", "alpha", "beta", "p_grow", "keep_forests")

_LE = {"u1": np.dtype("u1"), "u4": np.dtype("<u4"), "f4": np.dtype("<f4"), "f8": np.dtype("<f8"),
       "u2": np.dtype("<u2"), "i8": np.dtype("<i8")}


def _put(f: BinaryIO, a, code: str) -> None:
    f.write(np.ascontiguousarray(a, _LE[code]).tobytes())


def _get(f: BinaryIO, shape, code: str) -> np.ndarray:
    dt = _LE[code]
    count = int(np.prod(shape)) if len(shape) else 1
    raw = f.read(count * dt.itemsize)
    if len(raw) != count * dt.itemsize:
        raise ValueError("container truncated")
    return np.frombuffer(raw, dt).reshape(shape).copy()


def _nbytes(shape, code: str) -> int:
    return int(np.prod(shape)) * _LE[code].itemsize if len(shape) else _LE[code].itemsize


# ---------------------------------------------------------------- BFORGE1
def _put_forest_matrices(f: BinaryIO, forest: Forest) -> None:
    _put(f, forest.axis, "u4")
    _put(f, forest.cutpoint, "u4")
    _put(f, forest.leaf_value, "f4")


def _get_forest_matrices(f: BinaryIO, m: int, D: int, p: int) -> Forest:
    half, full = split_slots(D), heap_size(D)
    axis = _get(f, (m, half), "u4").astype(min_axis_dtype(p))
    cut = _get(f, (m, half), "u4").astype(np.uint8)
    leaf = _get(f, (m, full), "f4").astype(np.float32)
    return Forest(axis=axis, cutpoint=cut, leaf_value=leaf, max_depth=int(D))


def save_forest(f: BinaryIO, forest: Forest, grid: CutpointGrid) -> None:
    """BFORGE1: magic, (D, m, p) as uint32, per-axis cutpoint counts, the cutpoints
    (f64, axis by axis), then axis / cutpoint (uint32) and leaf values (f32)."""
    f.write(FOREST_MAGIC)
    f.write(struct.pack("<III", int(forest.max_depth), int(forest.axis.shape[0]), int(grid.n_axes)))
    _put(f, grid.counts, "u4")
    for cuts in grid.cutpoints:
        _put(f, cuts, "f8")
    _put_forest_matrices(f, forest)


def load_forest(f: BinaryIO) -> tuple[Forest, CutpointGrid]:
    magic = f.read(8)
    if magic != FOREST_MAGIC:
        raise ValueError(f"bad forest container magic {magic!r}")
    D, m, p = struct.unpack("<III", f.read(12))
    counts = _get(f, (p,), "u4")
    grid = CutpointGrid([_get(f, (int(c),), "f8") for c in counts])
    return _get_forest_matrices(f, m, D, p), grid


# ---------------------------------------------------------------- BFTRACE1
def _reference_config(config) -> dict:
    d = dataclasses.asdict(config)
    return {k: d[k] for k in REFERENCE_CONFIG_FIELDS}


class TraceFile:
    """BFTRACE1 writer with every section's offset fixed up front, so the
    arrays can arrive in any order and in pieces (kept draws chunk by chunk)."""

    def __init__(self, path: str, config, yscale, grid: CutpointGrid, n_train: int, n_iter: int,
                 n_test: Optional[int] = None, x_test: Optional[np.ndarray] = None, has_forests: bool = False):
        C, K, m, D = config.n_chains, config.n_kept, config.n_trees, config.max_depth
        self.C, self.K, self.m, self.D, self.n, self.n_test = C, K, m, D, int(n_train), n_test
        header = {
            "config": _reference_config(config),
            "center": yscale.center,
            "scale": yscale.scale,
            "sigma_shape": [C, K],
            "yhat_train_shape": [C, K, int(n_train)],
            "yhat_test_shape": None if n_test is None else [C, K, int(n_test)],
            "accepted_shape": [C, int(n_iter), m],
            "mean_leaves_shape": [C, K],
            "x_test_shape": None if x_test is None else list(x_test.shape),
            "grid_counts": [int(c) for c in grid.counts],
            "max_depth": D,
            "has_forests": bool(has_forests),
        }
        # this package's extra FitConfig fields, when not at their defaults (so a
        # trace of a default fit is byte-identical to the reference's file)
        defaults = {fl.name: fl.default for fl in dataclasses.fields(config)}
        extra = {k: v for k, v in dataclasses.asdict(config).items()
                 if k not in REFERENCE_CONFIG_FIELDS and v != defaults.get(k)}
        if extra:
            header["b200"] = {"config": extra}
        blob = json.dumps(header).encode()
        off = 8 + 8 + len(blob)
        self.off = {}
        for name, shape, code, present in (
                ("sigma", (C, K), "f8", True), ("yhat_train", (C, K, n_train), "f8", True),
                ("yhat_test", (C, K, n_test or 0), "f8", n_test is not None),
                ("accepted", (C, n_iter, m), "u1", True), ("mean_leaves", (C, K), "f8", True),
                ("x_test", tuple(x_test.shape) if x_test is not None else (0,), "f8", x_test is not None),
                ("grid", (int(np.sum(grid.counts)),), "f8", True)):
            if present:
                self.off[name] = off
                off += _nbytes(shape, code)
        self.tree_bytes = m * (4 * split_slots(D) * 2 + 4 * heap_size(D))
        if has_forests:
            self.off["forests"] = off
            off += C * K * self.tree_bytes
        self.size = off
        self.f = open(path, "wb")
        self.f.write(TRACE_MAGIC)
        self.f.write(struct.pack("<II", TRACE_VERSION, len(blob)))
        self.f.write(blob)
        self.f.truncate(self.size)
        self._at("grid", 0)
        for cuts in grid.cutpoints:
            _put(self.f, cuts, "f8")
        if x_test is not None:
            self._at("x_test", 0)
            _put(self.f, x_test, "f8")

    def _at(self, name: str, byte_offset: int) -> None:
        self.f.seek(self.off[name] + byte_offset)

    def write_sigma(self, sigma: np.ndarray) -> None:
        self._at("sigma", 0)
        _put(self.f, sigma, "f8")

    def write_accepted(self, accepted: np.ndarray) -> None:
        self._at("accepted", 0)
        _put(self.f, np.asarray(accepted).astype(np.uint8), "u1")

    def write_mean_leaves(self, mean_leaves: np.ndarray) -> None:
        self._at("mean_leaves", 0)
        _put(self.f, mean_leaves, "f8")

    def write_train_draws(self, chain: int, k0: int, draws: np.ndarray) -> None:
        """Kept draws k0 .. k0+len(draws) of one chain's training-row predictions."""
        self._at("yhat_train", ((chain * self.K + k0) * self.n) * 8)
        _put(self.f, draws, "f8")

    def write_test_draws(self, chain: int, k0: int, draws: np.ndarray) -> None:
        self._at("yhat_test", ((chain * self.K + k0) * self.n_test) * 8)
        _put(self.f, draws, "f8")

    def write_forest(self, chain: int, k: int, forest: Forest) -> None:
        self._at("forests", (chain * self.K + k) * self.tree_bytes)
        _put_forest_matrices(self.f, forest)

    def close(self) -> None:
        self.f.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def save_trace(path: str, trace) -> None:
    """Write a fit() trace as BFTRACE1 (needs the kept training-row draws:
    fit with keep_train_draws=True, or pass trace_path= to fit to stream them)."""
    if trace.yhat_train is None:
        raise ValueError("the trace holds no training-row draws (fit with keep_train_draws=True, "
                         "or fit(..., trace_path=...) to stream them from the device)")
    C, K, n = trace.yhat_train.shape
    n_test = None if trace.yhat_test is None else trace.yhat_test.shape[-1]
    with TraceFile(path, trace.config, trace.yscale, trace.grid, n, trace.accepted.shape[1], n_test,
                   trace.x_test, trace.forests is not None) as tf:
        tf.write_sigma(trace.sigma)
        tf.write_accepted(trace.accepted)
        tf.write_mean_leaves(trace.mean_leaves)
        for c in range(C):
            tf.write_train_draws(c, 0, trace.yhat_train[c])
            if n_test is not None:
                tf.write_test_draws(c, 0, trace.yhat_test[c])
            if trace.forests is not None:
                for k, forest in enumerate(trace.forests[c]):
                    tf.write_forest(c, k, forest)


def load_trace(path: str):
    """Read a BFTRACE1 container (written here or by the reference)."""
    from .regression import FitConfig, Trace, YScale
    with open(path, "rb") as f:
        magic = f.read(8)
        if magic != TRACE_MAGIC:
            raise ValueError(f"bad trace container magic {magic!r}")
        version, hlen = struct.unpack("<II", f.read(8))
        if version != TRACE_VERSION:
            raise ValueError(f"unsupported trace container version {version}")
        header = json.loads(f.read(hlen).decode())
        cfg = dict(header["config"])
        cfg.update(header.get("b200", {}).get("config", {}))
        known = {fl.name for fl in dataclasses.fields(FitConfig)}
        config = FitConfig(**{k: v for k, v in cfg.items() if k in known})
        sigma = _get(f, tuple(header["sigma_shape"]), "f8")
        yhat_train = _get(f, tuple(header["yhat_train_shape"]), "f8")
        yhat_test = None if header["yhat_test_shape"] is None else _get(f, tuple(header["yhat_test_shape"]), "f8")
        accepted = _get(f, tuple(header["accepted_shape"]), "u1").astype(bool)
        mean_leaves = _get(f, tuple(header["mean_leaves_shape"]), "f8")
        x_test = None if header["x_test_shape"] is None else _get(f, tuple(header["x_test_shape"]), "f8")
        grid = CutpointGrid([_get(f, (int(c),), "f8") for c in header["grid_counts"]])
        forests = None
        if header["has_forests"]:
            C, K = sigma.shape
            forests = [[_get_forest_matrices(f, config.n_trees, header["max_depth"], grid.n_axes) for _ in range(K)]
                       for _ in range(C)]
    return Trace(config=config, yscale=YScale(center=header["center"], scale=header["scale"]), grid=grid,
                 sigma=sigma, yhat_train=yhat_train, yhat_test=yhat_test, accepted=accepted,
                 mean_leaves=mean_leaves, forests=forests, x_test=x_test)


# ---------------------------------------------------------------- BFCKPT1
def save_checkpoint(path: str, state, hp) -> None:
    """Mid-chain checkpoint of a SamplerState: JSON header (shapes, iteration,
    sigma^2, hyperparameters, random stream) + forest, leaf-index cache (n, m),
    residuals (f32) and the quantized X / max_cuts / y the chain was built on."""
    from .sampler import DeviceRNG
    state.sync()
    forest = state.forest
    L = state.leaf_index
    resid = state.resid
    rng = state.rng
    if isinstance(rng, DeviceRNG):
        stream = {"kind": "device", "seed": int(rng.seed)}
    elif isinstance(rng, np.random.Generator):
        stream = {"kind": "numpy", "bit_generator": rng.bit_generator.state}
    else:
        raise TypeError("checkpoint needs a DeviceRNG or numpy Generator chain")
    header = {
        "version": CHECKPOINT_VERSION,
        "n": int(state.X.shape[0]), "p": int(state.X.shape[1]), "m": int(forest.axis.shape[0]),
        "max_depth": int(forest.max_depth), "iteration": int(state.iteration), "sigma2": float(state.sigma2),
        "hyperparams": dataclasses.asdict(hp), "rng": stream,
    }
    blob = json.dumps(header, default=int).encode()
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
        _put(f, state.X, "u1")
        _put(f, state.max_cuts, "i8")
        _put(f, state.y, "f4")
        _put(f, forest.axis.astype(np.uint16), "u2")
        _put(f, forest.cutpoint, "u1")
        _put(f, forest.leaf_value, "f4")
        _put(f, L, "u1")
        _put(f, resid, "f4")


def load_checkpoint(path: str, device: int = 0):
    """Rebuild the chain saved by save_checkpoint on `device`; returns (state, hp)."""
    from .sampler import DeviceRNG, Hyperparams, init_state
    with open(path, "rb") as f:
        if f.read(8) != CHECKPOINT_MAGIC:
            raise ValueError("bad checkpoint magic")
        (hlen,) = struct.unpack("<I", f.read(4))
        h = json.loads(f.read(hlen).decode())
        if h["version"] != CHECKPOINT_VERSION:
            raise ValueError(f"unsupported checkpoint version {h['version']}")
        n, p, m, D = h["n"], h["p"], h["m"], h["max_depth"]
        X = _get(f, (n, p), "u1")
        max_cuts = _get(f, (p,), "i8")
        y = _get(f, (n,), "f4")
        axis = _get(f, (m, split_slots(D)), "u2")
        cut = _get(f, (m, split_slots(D)), "u1")
        leaf = _get(f, (m, heap_size(D)), "f4")
        L = _get(f, (n, m), "u1")
        resid = _get(f, (n,), "f4")
    hp = Hyperparams(**h["hyperparams"])
    s = h["rng"]
    if s["kind"] == "device":
        rng = DeviceRNG(s["seed"])
    else:
        bg = getattr(np.random, s["bit_generator"]["bit_generator"])()
        bg.state = s["bit_generator"]
        rng = np.random.Generator(bg)
    state = init_state(X, max_cuts, y, hp, rng, device=device)
    state.restore(Forest(axis=axis.astype(min_axis_dtype(p)), cutpoint=cut, leaf_value=leaf, max_depth=D), L, resid,
                  h["sigma2"], h["iteration"])
    return state, hp

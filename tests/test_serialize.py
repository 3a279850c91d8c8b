"""BFORGE1 / BFTRACE1 containers (mirrors the reference's tests/test_serialize.py)
plus byte compatibility with files the reference itself wrote
(tests/golden/make_serialize_golden.py).  CPU only."""

import io
import struct
from pathlib import Path

import numpy as np
import pytest

from paper_2410_23244_b200 import serialize
from paper_2410_23244_b200.grid import CutpointGrid
from paper_2410_23244_b200.regression import FitConfig, Trace, YScale
from paper_2410_23244_b200.trees import Forest, serialized_tree_nbytes

from golden.make_serialize_golden import CONFIG, serialize_inputs

GOLD = Path(__file__).resolve().parent / "golden"


def _forest(t, D):
    return Forest(axis=t[0], cutpoint=t[1], leaf_value=t[2], max_depth=D)


def _trace(with_test: bool, **config_extra):
    a = serialize_inputs(with_test)
    return Trace(config=FitConfig(**CONFIG, **config_extra), yscale=YScale(center=a["center"], scale=a["scale"]),
                 grid=CutpointGrid(a["cuts"]), sigma=a["sigma"], yhat_train=a["yhat_train"],
                 yhat_test=a.get("yhat_test"), accepted=a["accepted"], mean_leaves=a["mean_leaves"],
                 forests=None if with_test else [[_forest(t, a["D"]) for t in ch] for ch in a["forests"]],
                 x_test=a.get("x_test"))


def _assert_trace_equal(a, b):
    assert a.config == b.config and a.yscale == b.yscale
    for k in ("sigma", "yhat_train", "accepted", "mean_leaves"):
        np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    for k in ("yhat_test", "x_test"):
        if getattr(a, k) is None:
            assert getattr(b, k) is None
        else:
            np.testing.assert_array_equal(getattr(a, k), getattr(b, k))
    for x, y in zip(a.grid.cutpoints, b.grid.cutpoints):
        np.testing.assert_array_equal(x, y)
    if a.forests is None:
        assert b.forests is None
    else:
        for ca, cb in zip(a.forests, b.forests):
            for fa, fb in zip(ca, cb):
                np.testing.assert_array_equal(fa.axis, fb.axis)
                np.testing.assert_array_equal(fa.cutpoint, fb.cutpoint)
                np.testing.assert_array_equal(fa.leaf_value, fb.leaf_value)


class TestForestContainer:
    def test_round_trip(self):
        a = serialize_inputs(False)
        forest, grid = _forest(a["forest"], a["D"]), CutpointGrid(a["cuts"])
        buf = io.BytesIO()
        serialize.save_forest(buf, forest, grid)
        buf.seek(0)
        got, got_grid = serialize.load_forest(buf)
        np.testing.assert_array_equal(got.axis, forest.axis)
        np.testing.assert_array_equal(got.cutpoint, forest.cutpoint)
        np.testing.assert_array_equal(got.leaf_value, forest.leaf_value)
        assert got.max_depth == forest.max_depth
        for x, y in zip(got_grid.cutpoints, grid.cutpoints):
            np.testing.assert_array_equal(x, y)

    def test_header_layout_and_payload(self):
        a = serialize_inputs(False)
        buf = io.BytesIO()
        serialize.save_forest(buf, _forest(a["forest"], a["D"]), CutpointGrid(a["cuts"]))
        raw = buf.getvalue()
        assert raw[:8] == b"BFORGE1\x00"
        assert struct.unpack_from("<III", raw, 8) == (3, 4, 2)
        assert np.frombuffer(raw, "<u4", count=2, offset=20).tolist() == [4, 3]
        grid_bytes = 8 + 12 + 4 * 2 + 8 * 7
        assert len(raw) - grid_bytes == 4 * serialized_tree_nbytes(3)

    def test_matches_reference_bytes(self):
        """The reference's save_forest output, byte for byte, both ways."""
        ref = (GOLD / "ref_forest.bforge").read_bytes()
        forest, grid = serialize.load_forest(io.BytesIO(ref))
        a = serialize_inputs(False)
        np.testing.assert_array_equal(forest.leaf_value, a["forest"][2])
        buf = io.BytesIO()
        serialize.save_forest(buf, forest, grid)
        assert buf.getvalue() == ref

    def test_rejects_bad_magic(self):
        with pytest.raises(ValueError, match="magic"):
            serialize.load_forest(io.BytesIO(b"NOTMAGIC" + b"\0" * 64))


class TestTraceContainer:
    @pytest.mark.parametrize("with_test", [False, True])
    def test_round_trip(self, tmp_path, with_test):
        trace = _trace(with_test)
        serialize.save_trace(str(tmp_path / "t.bin"), trace)
        _assert_trace_equal(trace, serialize.load_trace(str(tmp_path / "t.bin")))

    @pytest.mark.parametrize("with_test,name", [(False, "ref_trace.bftrace"), (True, "ref_trace_test.bftrace")])
    def test_matches_reference_bytes(self, tmp_path, with_test, name):
        """Reads what the reference wrote; writes the same bytes back (config = the reference's fields)."""
        ref = GOLD / name
        _assert_trace_equal(_trace(with_test), serialize.load_trace(str(ref)))
        serialize.save_trace(str(tmp_path / "t.bin"), _trace(with_test))
        assert (tmp_path / "t.bin").read_bytes() == ref.read_bytes()

    def test_extra_config_fields_survive_and_stay_out_of_config(self, tmp_path):
        trace = _trace(False, rng="host", keep_train_draws=True)
        path = tmp_path / "t.bin"
        serialize.save_trace(str(path), trace)
        raw = path.read_bytes()
        hlen = struct.unpack_from("<I", raw, 12)[0]
        import json
        header = json.loads(raw[16:16 + hlen])
        assert list(header["config"]) == list(serialize.REFERENCE_CONFIG_FIELDS)
        assert header["b200"]["config"]["rng"] == "host"
        assert serialize.load_trace(str(path)).config == trace.config

    def test_pieces_equal_whole(self, tmp_path):
        """TraceFile fed out of order, draws in chunks (as fit streams them) == save_trace."""
        trace = _trace(False)
        serialize.save_trace(str(tmp_path / "whole.bin"), trace)
        C, K, n = trace.yhat_train.shape
        with serialize.TraceFile(str(tmp_path / "pieces.bin"), trace.config, trace.yscale, trace.grid, n,
                                 trace.accepted.shape[1], None, None, True) as tf:
            for c in reversed(range(C)):
                for k in range(K):
                    tf.write_forest(c, k, trace.forests[c][k])
                tf.write_train_draws(c, 2, trace.yhat_train[c, 2:])
                tf.write_train_draws(c, 0, trace.yhat_train[c, :2])
            tf.write_mean_leaves(trace.mean_leaves)
            tf.write_accepted(trace.accepted)
            tf.write_sigma(trace.sigma)
        assert (tmp_path / "pieces.bin").read_bytes() == (tmp_path / "whole.bin").read_bytes()

    def test_needs_draws(self, tmp_path):
        trace = _trace(False)
        trace.yhat_train = None
        with pytest.raises(ValueError, match="draws"):
            serialize.save_trace(str(tmp_path / "t.bin"), trace)

    def test_rejects_bad_magic(self, tmp_path):
        path = tmp_path / "bad.bin"
        path.write_bytes(b"WRONG!!!" + b"\0" * 32)
        with pytest.raises(ValueError, match="magic"):
            serialize.load_trace(str(path))

"""CPU: the native BAL input path (include/povar_bal.h) against the reference's own
parse_bal / write_bal / prune_underobserved outputs (tests/golden/bal_cases.json,
tiny.bal.gz, prune.npz from tests/golden/make_golden.py).  Host-only code: no GPU."""

import bz2
import gzip
import io
import json

import numpy as np
import pytest

from _pvutil import GOLDEN, reference_stratba
from paper_2405_05079_b200 import bal, synth

CASES = json.loads((GOLDEN / "bal_cases.json").read_text())


def _check(case, parse):
    if "error" in case:
        with pytest.raises(bal.BalParseError) as ei:
            parse(case["text"])
        assert [ei.value.line, str(ei.value)] == case["error"], case["name"]
        return
    p = parse(case["text"])
    ok = case["ok"]
    assert [p.num_cameras, p.num_landmarks, p.num_observations] == ok["n"]
    assert p.camera_indices.tolist() == ok["cam"]
    assert p.landmark_indices.tolist() == ok["pt"]
    for got, want in ((p.measurements, ok["meas"]), (p.metric_cameras, ok["cams"]),
                      (p.metric_points, ok["pts"])):
        assert [[repr(float(v)) for v in r] for r in got] == want, case["name"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_parse_matches_reference(case):
    _check(case, lambda t: bal.parse_bal(io.StringIO(t)))


@pytest.mark.parametrize("threads", [2, 3, 8])
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_parse_chunked_matches_reference(case, threads):
    """Forced multi-chunk parses (64-byte chunks) give the same arrays / first error."""
    _check(case, lambda t: bal.parse_bytes(t.encode("utf-8"), n_threads=threads))


def test_tiny_file_written_by_reference_round_trips():
    pr, _ = synth.make_problem("tiny", 0)
    for threads in (0, 1, 7):
        got = bal.parse_bytes(gzip.decompress((GOLDEN / "tiny.bal.gz").read_bytes()), threads)
        np.testing.assert_array_equal(got.camera_indices, pr.camera_indices)
        np.testing.assert_array_equal(got.landmark_indices, pr.landmark_indices)
        np.testing.assert_array_equal(got.measurements, pr.measurements)  # .17g lossless
    assert bal.load_bal(GOLDEN / "tiny.bal.gz").num_observations == pr.num_observations


@pytest.mark.parametrize("codec", ["plain", "gzip", "bz2"])
def test_write_load_round_trip(tmp_path, codec):
    stratba = reference_stratba()  # the reference's own writer (bal_io.py:206-226)
    pr, _ = synth.make_problem("small", 0)
    buf = io.StringIO()
    stratba.bal_io.write_bal(pr, buf)
    data = buf.getvalue().encode()
    path = tmp_path / "p.bal"
    path.write_bytes({"plain": lambda d: d, "gzip": gzip.compress,
                      "bz2": bz2.compress}[codec](data))
    got = bal.load_bal(path)
    np.testing.assert_array_equal(got.camera_indices, pr.camera_indices)
    np.testing.assert_array_equal(got.landmark_indices, pr.landmark_indices)
    np.testing.assert_array_equal(got.measurements, pr.measurements)
    assert not got.metric_cameras.any() and not got.metric_points.any()
    one = bal.parse_bytes(data, n_threads=1)
    many = bal.parse_bytes(data, n_threads=8)
    np.testing.assert_array_equal(one.measurements, many.measurements)
    np.testing.assert_array_equal(one.landmark_indices, many.landmark_indices)


def test_prune_matches_reference():
    from paper_2405_05079_b200.types import BaProblem
    z = np.load(GOLDEN / "prune.npz")
    raw = BaProblem(7, 40, len(z["cam_idx"]), z["cam_idx"], z["lm_idx"], z["meas"], z["cams"],
                    z["pts"])
    p = bal.prune_underobserved(raw)
    assert [p.num_cameras, p.num_landmarks, p.num_observations] == z["p_n"].tolist()
    np.testing.assert_array_equal(p.camera_indices, z["p_cam"])
    np.testing.assert_array_equal(p.landmark_indices, z["p_lm"])
    np.testing.assert_array_equal(p.measurements, z["p_meas"])
    np.testing.assert_array_equal(p.metric_cameras, z["p_cams"])
    np.testing.assert_array_equal(p.metric_points, z["p_pts"])
    # nothing to prune -> the same object (bal_io.py:261-262)
    assert bal.prune_underobserved(p) is p

"""CPU: host logic of the pipeline caller (pipeline.py:34-141 of the reference) and
the trace-CSV artifacts (evaluation.py:154-200), against the reference's own
artifacts in tests/golden/pipeline_*."""

import io

import numpy as np
import pytest

from _pvutil import GOLDEN
from paper_2405_05079_b200 import evaluation, pipeline
from paper_2405_05079_b200.types import ConvergenceTrace, ProjectiveState, TraceRecord


def test_runspec_validation_and_configs():
    spec = pipeline.RunSpec(inputs=[], stage1_solver="iterative", stage2_solver="ripcg")
    spec.validate()
    c1, c2 = spec.stage1_config(), spec.stage2_config()
    assert (c1.mode, c1.inner_solver, c2.mode, c2.inner_solver) == ("varpro", "pcg", "joint",
                                                                      "pcg")
    assert pipeline.RunSpec(inputs=[], stage1_solver="poba").stage1_config().mode == "joint"
    for bad in (dict(stage="nope"), dict(stage1_solver="x"), dict(stage2_solver="y"),
                dict(max_iterations=0), dict(eta=1.5)):
        with pytest.raises(ValueError):
            pipeline.RunSpec(inputs=[], **bad).validate()
    echo = pipeline.RunSpec(inputs=[], seed=3, max_iterations=10).config_echo()
    assert echo == {"seed": 3, "stage": "full", "stage1_solver": "povar",
                    "stage2_solver": "ripoba", "eta": 0.1, "initial_lambda": 1e-4,
                    "max_iterations": 10, "function_tolerance": 1e-6, "power_order": 20,
                    "power_threshold": 0.01, "inner_iterations": 500}


def test_reference_trace_csv_round_trips():
    for tag in ("povar", "iterative"):
        text = (GOLDEN / f"pipeline_{tag}_trace.csv").read_text()
        traces = evaluation.read_trace_csv(io.StringIO(text))
        assert [t.stage for t in traces] == (["stage1", "stage2", "full"] if tag == "povar"
                                             else ["stage1"])
        out = io.StringIO()
        evaluation.write_trace_csv(traces, out)
        assert out.getvalue().replace("\r\n", "\n") == text.replace("\r\n", "\n")
    with pytest.raises(ValueError):
        evaluation.read_trace_csv(io.StringIO("a,b\n"))


def test_full_trace_convention():
    s2 = ConvergenceTrace("ripoba", "p", "stage2",
                          [TraceRecord(0, 5.0, 0.0), TraceRecord(1, 4.0, 0.5)], 5.0)
    ft = pipeline.full_trace(9.0, 2.0, s2)
    assert ft.stage == "full" and ft.initial_cost == 9.0
    assert [(r.iteration, r.cost, r.elapsed_seconds) for r in ft.records] == [
        (0, 9.0, 0.0), (1, 5.0, 2.0), (2, 4.0, 2.5)]


def test_state_file_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    st = ProjectiveState(rng.standard_normal((3, 3, 4)), rng.standard_normal((5, 4)))
    pipeline.write_state(st, tmp_path / "s.txt")
    back = pipeline.read_state(tmp_path / "s.txt")
    np.testing.assert_array_equal(back.cameras, st.cameras)
    np.testing.assert_array_equal(back.landmarks, st.landmarks)

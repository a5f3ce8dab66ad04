"""GPU: the pipeline caller end to end (BAL file -> prune -> random_init -> stage 1 ->
lift -> stage 2 -> artifacts) against the reference's run_problem artifacts on the
same file (tests/golden/pipeline_*, made from tiny.bal.gz by make_golden.py).
Power-series runs: costs within north_star's 1e-6 LM-trace tolerance, counts and
config identical (seed 0, 30 iterations: a chain the CPU oracle reproduces within
3e-11).  PCG runs: stage 1 only, within 1e-5 -- each CG step is accurate to its
pcg_tolerance (1e-6), which the LM trace inherits."""

import json

import numpy as np
import pytest

from _pvutil import GOLDEN, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag,stage,s1,s2,its,tol", [
    ("povar", "full", "povar", "ripoba", 30, 1e-6),
    ("iterative", "stage1", "iterative", "ripcg", 20, 1e-5)])
def test_run_problem_matches_reference(tmp_path, tag, stage, s1, s2, its, tol):
    from paper_2405_05079_b200 import evaluation, pipeline
    spec = pipeline.RunSpec(inputs=[str(GOLDEN / "tiny.bal.gz")], seed=0, stage=stage,
                            stage1_solver=s1, stage2_solver=s2, max_iterations=its,
                            out_dir=str(tmp_path))
    summary = pipeline.run_problem(GOLDEN / "tiny.bal.gz", spec)
    want = json.loads((GOLDEN / f"pipeline_{tag}_summary.json").read_text())
    for k in ("schema_version", "problem_id", "num_cameras", "num_landmarks",
              "num_observations", "pruned_landmarks", "config"):
        assert summary[k] == want[k], k
    assert sorted(summary["stages"]) == sorted(want["stages"])
    for st in want["stages"]:
        got, ref = summary["stages"][st], want["stages"][st]
        assert got["solver"] == ref["solver"] and got["iterations"] == ref["iterations"]
        for k in ("initial_cost", "final_cost") + (("pre_stage1_cost",) if st == "stage2"
                                                    else ()):
            assert rel(got[k], ref[k]) <= tol, (st, k)
    ours = evaluation.read_trace_csv(tmp_path / "tiny_trace.csv")
    ref = evaluation.read_trace_csv(GOLDEN / f"pipeline_{tag}_trace.csv")
    assert [(t.solver_id, t.stage, len(t.records)) for t in ours] == \
        [(t.solver_id, t.stage, len(t.records)) for t in ref]
    for a, b in zip(ours, ref):
        ca = np.array([r.cost for r in a.records])
        cb = np.array([r.cost for r in b.records])
        assert rel(ca, cb) <= tol, a.stage
        assert [y < x for x, y in zip(ca, ca[1:])] == [y < x for x, y in zip(cb, cb[1:])]
    assert (tmp_path / "tiny_state.txt").exists() and (tmp_path / "tiny_summary.json").exists()

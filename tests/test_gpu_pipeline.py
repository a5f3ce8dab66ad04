"""GPU: the reference's OWN caller around the hot path, switched onto the device.

``stratba.pipeline.run_problem`` (pipeline.py:144-247, the unmodified reference installed
under baseline/_ref) runs BAL file -> prune -> random_init -> stage 1 -> lift -> stage 2
-> artifacts with its ``lm_minimize`` (and, for the povar chain, ``random_init``) rebound
to the device path by ``paper_2405_05079_b200.integration.enable`` -- the INTEGRATION.md
section 1 switch.  Its artifacts are compared with those the reference wrote on the same
file on its CPU path (tests/golden/pipeline_*, make_golden.py).  Power-series runs: costs
within north_star's 1e-6 LM-trace tolerance, counts and config identical (seed 0, 30
iterations: a chain the CPU oracle reproduces within 3e-11).  PCG runs: stage 1 only,
within 1e-5 -- each CG step is accurate to its pcg_tolerance (1e-6), which the LM trace
inherits."""

import json

import numpy as np
import pytest

from _pvutil import GOLDEN, reference_stratba, rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("tag,stage,s1,s2,its,tol,dev_init", [
    ("povar", "full", "povar", "ripoba", 30, 1e-6, True),
    ("iterative", "stage1", "iterative", "ripcg", 20, 1e-5, False)])
def test_reference_run_problem_on_device(tmp_path, tag, stage, s1, s2, its, tol, dev_init):
    stratba = reference_stratba()
    from paper_2405_05079_b200 import integration, solver
    calls = []
    real = solver.lm_minimize

    def counting(*a, **k):
        calls.append(a[2])
        return real(*a, **k)

    integration.enable(stratba, random_init=dev_init)
    solver.lm_minimize = counting  # the dispatcher resolves solver.lm_minimize at call time
    try:
        spec = stratba.pipeline.RunSpec(inputs=[str(GOLDEN / "tiny.bal.gz")], seed=0,
                                        stage=stage, stage1_solver=s1, stage2_solver=s2,
                                        max_iterations=its, out_dir=str(tmp_path))
        summary = stratba.pipeline.run_problem(GOLDEN / "tiny.bal.gz", spec)
    finally:
        solver.lm_minimize = real
        integration.disable()
    assert calls == ([1, 2] if stage == "full" else [1])  # every stage ran on the device
    assert stratba.pipeline.lm_minimize is stratba.solvers.lm_minimize  # restored
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
    read = stratba.evaluation.read_trace_csv
    ours = read(tmp_path / "tiny_trace.csv")
    ref = read(GOLDEN / f"pipeline_{tag}_trace.csv")
    assert [(t.solver_id, t.stage, len(t.records)) for t in ours] == \
        [(t.solver_id, t.stage, len(t.records)) for t in ref]
    worst = 0.0
    for a, b in zip(ours, ref):
        ca = np.array([r.cost for r in a.records])
        cb = np.array([r.cost for r in b.records])
        worst = max(worst, float(np.max(np.abs(ca - cb) / np.abs(cb))))
        assert rel(ca, cb) <= tol, a.stage
        assert [y < x for x, y in zip(ca, ca[1:])] == [y < x for x, y in zip(cb, cb[1:])]
    print(f"pipeline {tag}: max relative cost difference {worst:.2e}")
    assert (tmp_path / "tiny_state.txt").exists() and (tmp_path / "tiny_summary.json").exists()


def test_direct_inner_solver_stays_on_the_reference():
    """inner_solver="direct" is not on the GPU path: the switch hands it back to the
    reference instead of failing or falling back silently."""
    stratba = reference_stratba()
    from paper_2405_05079_b200 import integration
    from _pvutil import golden
    z = golden("mini_0.npz")
    p = stratba.BaProblem(int(z["n_cameras"]), int(z["n_landmarks"]), len(z["cam_idx"]),
                          z["cam_idx"].astype(np.int64), z["lm_idx"].astype(np.int64),
                          z["meas"])
    st = stratba.ProjectiveState(z["cams"], z["lms"])
    cfg = stratba.SolverConfig(max_outer_iterations=3, inner_solver="direct")
    want = stratba.solvers.lm_minimize(p, st, 1, cfg)[1]
    integration.enable(stratba)
    try:
        got = stratba.solvers.lm_minimize(p, st, 1, cfg)[1]
    finally:
        integration.disable()
    assert [r.cost for r in got.records] == [r.cost for r in want.records]

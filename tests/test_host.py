"""CPU: host-side logic, API types, the C-ABI library surface and the generator."""

import ast
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_solver_config_validation_mirrors_reference():
    from paper_2405_05079_b200 import SolverConfig, PoseConfig
    cfg = SolverConfig()
    assert (cfg.max_outer_iterations, cfg.function_tolerance, cfg.initial_lambda,
            cfg.max_power_order, cfg.power_threshold, cfg.max_inner_iterations,
            cfg.pose.eta) == (50, 1e-6, 1e-4, 20, 0.01, 500, 0.1)
    for bad in (dict(inner_solver="magic"), dict(mode="alternation"),
                dict(initial_lambda=0.0), dict(max_power_order=-1)):
        with pytest.raises(ValueError):
            SolverConfig(**bad)
    with pytest.raises(ValueError):
        PoseConfig(1.5)


def test_problem_and_state_validation():
    from paper_2405_05079_b200 import BaProblem, ProjectiveState
    with pytest.raises(ValueError):
        BaProblem(2, 1, 1, np.array([2]), np.array([0]), np.zeros((1, 2)))
    with pytest.raises(ValueError):
        BaProblem(2, 1, 2, np.array([0]), np.array([0]), np.zeros((1, 2)))
    with pytest.raises(ValueError):
        ProjectiveState(np.zeros((2, 4, 3)), np.zeros((1, 4)))
    p = BaProblem(2, 1, 1, np.array([1]), np.array([0]), np.zeros((1, 2)))
    assert not p.measurements.flags.writeable


def test_trace_and_labels():
    from paper_2405_05079_b200 import ConvergenceTrace, SolverConfig, TraceRecord, solver_label
    with pytest.raises(ValueError):
        ConvergenceTrace("a", "p", "stage1", [TraceRecord(0, 1.0, 0.0), TraceRecord(1, 0.5, -1)],
                         1.0)
    assert solver_label(1, SolverConfig()) == "povar"
    assert solver_label(1, SolverConfig(mode="joint")) == "poba"
    assert solver_label(2, SolverConfig()) == "ripoba"


def test_header_symbols_are_bound_and_exported():
    """Every entry point declared in include/*.h is exported by libpovar.so and bound."""
    from paper_2405_05079_b200 import _lib
    header = "".join(p.read_text() for p in sorted((ROOT / "include").glob("*.h")))
    declared = set(re.findall(r"\b(pv_[a-z_0-9]+)\s*\(", header))
    bound = {name for name, _, _ in _lib.SIGNATURES}
    assert declared == bound, declared ^ bound
    lib = _lib.load()  # loading needs no GPU
    for name in declared:
        assert hasattr(lib, name), name


def test_no_cpu_fallback_without_gpu():
    import torch

    import paper_2405_05079_b200 as pv
    from paper_2405_05079_b200 import synth
    if torch.cuda.is_available():
        pytest.skip("a GPU is present; the loud-failure path is exercised on CPU hosts")
    pr, _ = synth.make_problem("tiny", 0)
    with pytest.raises(RuntimeError):
        pv.DeviceProblem(pr, 0.1)


def test_product_package_never_imports_the_oracle():
    pkg = ROOT / "paper_2405_05079_b200"
    for path in pkg.rglob("*.py"):
        tree = ast.parse(path.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                names = [a.name for a in node.names]
            elif isinstance(node, ast.ImportFrom):
                names = [node.module or ""]
            else:
                continue
            assert not any(n.split(".")[0] == "oracle" for n in names), path


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan_tiles_and_balances(world):
    from paper_2405_05079_b200 import shard, synth
    pr, _ = synth.make_problem("small", 0)
    plan = shard.plan_shards(pr, world)
    assert plan[0][0] == 0 and plan[-1][1] == pr.num_landmarks
    assert all(a[1] == b[0] for a, b in zip(plan, plan[1:]))
    counts = shard.shard_observation_counts(pr, plan)
    assert sum(counts) == pr.num_observations
    ideal = pr.num_observations / world
    assert max(counts) - ideal <= 64  # one landmark's worth of slack


@pytest.mark.parametrize("name", ["tiny", "small"])
def test_generator_matches_config(name):
    from paper_2405_05079_b200 import synth
    cfg = synth.CONFIGS[name]
    pr, truth = synth.make_problem(name, 0)
    assert (pr.num_cameras, pr.num_landmarks) == (cfg.n_cameras, cfg.n_landmarks)
    k = np.bincount(pr.landmark_indices, minlength=pr.num_landmarks)
    assert k.min() >= 2
    if name == "tiny":
        assert k.max() <= 6
    pairs = pr.camera_indices * pr.num_landmarks + pr.landmark_indices
    assert len(np.unique(pairs)) == pr.num_observations  # distinct cameras per landmark
    # noise-free ground truth reproduces the measurements to ~1 px / mean focal
    gt = synth.ground_truth_state(truth)
    u = np.einsum("nij,nj->ni", gt.cameras[pr.camera_indices], gt.landmarks[pr.landmark_indices])
    assert np.all(u[:, 2] > 0)
    err = np.abs(u[:, :2] / u[:, 2:] - pr.measurements).max() * truth["focal_mean"]
    assert err < 6.0
    # deterministic
    pr2, _ = synth.make_problem(name, 0)
    np.testing.assert_array_equal(pr.measurements, pr2.measurements)


def test_retract_and_lift():
    import paper_2405_05079_b200 as pv
    st = pv.ProjectiveState(np.arange(24.0).reshape(2, 3, 4) + 1, np.ones((3, 4)))
    r = pv.lift_stage1_to_stage2(st)
    np.testing.assert_allclose(np.linalg.norm(r.cameras.reshape(-1, 12), axis=1), 1.0)
    np.testing.assert_allclose(np.linalg.norm(r.landmarks, axis=1), 1.0)
    with pytest.raises(ValueError):
        pv.retract(pv.ProjectiveState(np.zeros((1, 3, 4)), np.ones((1, 4))))


def test_integration_switch_rebinds_and_restores():
    """integration.enable rebinds the reference's lm_minimize (solvers + pipeline namespaces,
    pipeline.py:18) and optionally random_init; disable restores them (no GPU call)."""
    from _pvutil import reference_stratba
    from paper_2405_05079_b200 import integration, solver
    stratba = reference_stratba()
    ref_lm, ref_init = stratba.solvers.lm_minimize, stratba.pipeline.random_init
    integration.enable(stratba, random_init=True)
    try:
        assert stratba.pipeline.lm_minimize is stratba.solvers.lm_minimize is not ref_lm
        assert stratba.pipeline.random_init is solver.random_init
        assert stratba.bal_io.random_init is solver.random_init
    finally:
        integration.disable()
    assert stratba.solvers.lm_minimize is ref_lm and stratba.pipeline.lm_minimize is ref_lm
    assert stratba.pipeline.random_init is ref_init


def test_stage2_rejects_non_unit_state_before_any_device_work():
    """riemannian.py:46-48: the tangent basis needs unit vectors.  The check runs on the
    host before the device is touched, with the reference's message (tests/golden/degen.npz
    holds the reference's own exception text)."""
    from _pvutil import golden
    from paper_2405_05079_b200 import solver
    from paper_2405_05079_b200.types import ProjectiveState
    z = golden("degen.npz")
    st = ProjectiveState(z["cams"], z["lms"])
    with pytest.raises(ValueError) as ei:
        solver._check_unit(st)
    assert str(ei.value) == str(z["nonunit_message"])
    cams = st.cameras.reshape(len(st.cameras), 12)
    unit = ProjectiveState((cams / np.linalg.norm(cams, axis=1)[:, None]).reshape(-1, 3, 4),
                           st.landmarks / np.linalg.norm(st.landmarks, axis=1)[:, None])
    solver._check_unit(unit)
    bad = np.array(unit.landmarks)
    bad[3] *= 1.0 + 2e-9  # beyond UNIT_TOL = 1e-9 (riemannian.py:26)
    with pytest.raises(ValueError):
        solver._check_unit(ProjectiveState(unit.cameras, bad))


def test_householder_bases_match_reference_convention():
    """riemannian_step's bases argument is validated against the Householder construction
    (riemannian.py:37-56) the device applies implicitly."""
    from _pvutil import reference_stratba
    from paper_2405_05079_b200 import solver
    from paper_2405_05079_b200.types import ProjectiveState
    stratba = reference_stratba()
    rng = np.random.default_rng(4)
    cams = rng.standard_normal((5, 12))
    cams[0, 0] = -abs(cams[0, 0])
    cams /= np.linalg.norm(cams, axis=1)[:, None]
    lms = rng.standard_normal((9, 4))
    lms /= np.linalg.norm(lms, axis=1)[:, None]
    st = ProjectiveState(cams.reshape(5, 3, 4), lms)
    ref = stratba.riemannian.state_tangent_bases(st)
    np.testing.assert_allclose(solver._householder_bases(cams), ref.camera_bases, atol=1e-15)
    solver._check_bases(st, ref)
    other = stratba.riemannian.TangentBasis(ref.camera_bases[:, :, ::-1].copy(),
                                            ref.landmark_bases)
    with pytest.raises(ValueError):
        solver._check_bases(st, other)


def test_merge_states_and_loopback_id():
    """shard.merge_states: replicated cameras of rank 0 + each rank's own landmark range;
    pv_loopback_id (host-only) returns a 128-byte id tagged as an in-process group."""
    from paper_2405_05079_b200 import shard
    from paper_2405_05079_b200.types import ProjectiveState
    rng = np.random.default_rng(3)
    cams = rng.standard_normal((4, 3, 4))
    base = rng.standard_normal((10, 4))
    plan = [(0, 3), (3, 7), (7, 10)]
    states = []
    for r, (b, e) in enumerate(plan):
        lms = base.copy()
        lms[b:e] += r + 1.0
        states.append(ProjectiveState(cams, lms))
    merged = shard.merge_states(states, plan)
    want = base.copy()
    for r, (b, e) in enumerate(plan):
        want[b:e] += r + 1.0
    np.testing.assert_array_equal(merged.landmarks, want)
    np.testing.assert_array_equal(merged.cameras, cams)
    lid = shard.loopback_id(3)
    assert len(lid) == 128 and lid[:8] == (0x4b4250504f4f4c50).to_bytes(8, "little")

"""CUDA PCG inner solver (solvers.py:153-187) vs the reference's fixtures
(tests/golden/pcg.npz) and the oracle (needs a B200).

Parity rules: the exact Schur block diagonal within 1e-12 of ||U|| (it is a
cancellation U - sum W V+ W^T); CG results by ``check_pcg_result``
(test_oracle_pcg.py): identical iteration counts and flags, updates within
max(1e-9, 5 % of the solve's own error); LM traces within north_star's 1e-6
with the same accept/reject sequence.
"""

import numpy as np
import pytest

import _kat
from _pvutil import golden, problem_from, rel
from oracle import povar_oracle as O
from test_oracle_pcg import SETTINGS, check_pcg_result, systems

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pv():
    import paper_2405_05079_b200 as pv
    return pv


@pytest.fixture(scope="module")
def pcgz():
    return golden("pcg.npz")


CASES = [("s1v_", 1, 1e-4, "pose_only"), ("s1j_", 1, 0.3, "both"), ("s2_", 2, 1e-3, "both")]


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("tag,stage,lam,mode", CASES)
def test_pcg_matches_reference(pv, pcgz, seed, tag, stage, lam, mode):
    from paper_2405_05079_b200 import _lib
    _, z, osys = systems(seed)
    s = osys[tag]
    pr = problem_from(z)
    dp = pv.DeviceProblem(pr, 0.1)
    st = pv.ProjectiveState(z["cams"], z["lms"]) if stage == 1 else \
        pv.ProjectiveState(z["cams2"], z["lms2"])
    sysm = pv.assemble_system(pr, st, stage, lam, mode, dp=dp)
    pre = f"m{seed}_{tag}"
    d = 12 if stage == 1 else 11
    x_dense = np.linalg.solve(O.dense_reduced_matrix(s), O.schur_rhs(s))
    for st_tag, tol, cap in SETTINGS:
        rep = pv.pcg_schur_solve(sysm, pv.SolverConfig(pcg_tolerance=tol, max_inner_iterations=cap,
                                                       inner_solver="pcg"))
        assert rep.power_order_used == 0
        check_pcg_result(rep.pose_update, rep.landmark_update, rep.inner_iterations_used,
                         rep.truncation_estimate, rep.flag, pcgz, pre, st_tag, tol, cap, x_dense)
    n_p = dp.n_p
    sd = dp.debug(_lib.PV_DBG_SDIAG).reshape(n_p, 12, 12)[:, :d, :d]
    assert np.linalg.norm(sd - pcgz[pre + "diag"]) <= 1e-12 * np.linalg.norm(s.U)
    mi = dp.debug(_lib.PV_DBG_MINV).reshape(n_p, 12, 12)[:, :d, :d]
    assert rel(mi, np.linalg.inv(pcgz[pre + "diag"])) <= 1e-9


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("stage", [1, 2])
def test_pcg_lm_traces(pv, pcgz, seed, stage):
    z = golden(f"mini_{seed}.npz")
    pr = problem_from(z)
    st = pv.ProjectiveState(z["cams"], z["lms"]) if stage == 1 else \
        pv.ProjectiveState(z["cams2"], z["lms2"])
    cfg = pv.SolverConfig(max_outer_iterations=10, inner_solver="pcg")
    _, trace = pv.lm_minimize(pr, st, stage, cfg)
    assert trace.solver_id == ("iterative" if stage == 1 else "ripcg")
    costs = np.array([r.cost for r in trace.records])
    want = pcgz[f"m{seed}_lm{stage}_costs"]
    assert len(costs) == len(want)
    assert [b < a for a, b in zip(costs, costs[1:])] == [b < a for a, b in zip(want, want[1:])]
    assert rel(costs, want) <= 1e-6


def test_pcg_tiny_trace(pv, pcgz):
    from paper_2405_05079_b200 import synth
    pr, _ = synth.make_problem("tiny", 0)
    st = synth.random_state(pr, 1)
    _, trace = pv.lm_minimize(pr, st, 1, pv.SolverConfig(max_outer_iterations=20,
                                                         inner_solver="pcg"))
    costs = np.array([r.cost for r in trace.records])
    want = pcgz["tiny_lm1_costs"]
    assert len(costs) == len(want)
    assert rel(costs, want) <= 1e-6


def test_pcg_known_answers(pv):
    """test_solvers.py:112-126: perfect preconditioner (no coupling) -> one iteration;
    zero RHS -> zero pose update after 0 iterations; an iteration cap of 0 -> rel 1."""
    pr, st = _kat.uncoupled_case()
    sysm = pv.assemble_system(pr, st, 1, 0.3, "pose_only")
    rep = pv.pcg_schur_solve(sysm, pv.SolverConfig(pcg_tolerance=1e-6))
    assert rep.inner_iterations_used == 1
    g = O.graph_of(pr)
    ref = O.pcg_solve(O.assemble(g, O.linearize(g, st.cameras, st.landmarks, 1), 0.3, False),
                      500, 1e-6)
    assert ref.iterations == 1
    assert rel(rep.pose_update, ref.pose_update) <= 1e-12
    its, rel0, flag = sysm.dp.pcg_solve(0, 1e-6)  # below SolverConfig's range: raw call
    assert (its, rel0, flag) == (0, 1.0, None)
    assert not sysm.dp.step(1)[0].any()
    pr, st = _kat.affine_consistent_case()
    sysm = pv.assemble_system(pr, st, 1, 1e-4, "pose_only")
    rep = pv.pcg_schur_solve(sysm, pv.SolverConfig())
    assert rep.inner_iterations_used == 0 and rep.truncation_estimate == 0.0
    assert not rep.pose_update.any()


@pytest.mark.parametrize("stage", [1, 2])
def test_pcg_collective_path_and_blocking(pv, stage):
    """Sharded code path over a 1-rank NCCL communicator reproduces the fused PCG bit
    for bit (fixed-order reductions); several landmark blocks change only the
    summation order of S'.p (compared over a fixed 12 iterations)."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    pr = problem_from(z)
    st = pv.ProjectiveState(z["cams"], z["lms"]) if stage == 1 else \
        pv.ProjectiveState(z["s2_cams0"], z["s2_lms0"])
    outs = []
    for forced, block_bytes in ((0, 1 << 30), (1, 1 << 30), (0, 64 << 10)):
        dp = pv.DeviceProblem(pr, 0.1)
        dp.set_option(_lib.PV_OPT_BLOCK_BYTES, block_bytes)
        dp.set_option(_lib.PV_OPT_FORCE_COLLECTIVE, forced)
        sysm = pv.assemble_system(pr, st, stage, 1e-3, "both" if stage == 2 else "pose_only",
                                  dp=dp)
        rep = pv.pcg_schur_solve(sysm, pv.SolverConfig(pcg_tolerance=1e-300,
                                                       max_inner_iterations=12))
        outs.append((dp.info()["blocks"], rep))
    assert outs[0][0] == 1 and outs[2][0] > 1
    a, b, c = (o[1] for o in outs)
    assert a.inner_iterations_used == b.inner_iterations_used
    np.testing.assert_array_equal(a.pose_update, b.pose_update)
    np.testing.assert_array_equal(a.landmark_update, b.landmark_update)
    # blocking changes the summation order of y only
    assert a.inner_iterations_used == c.inner_iterations_used == 12
    assert rel(c.pose_update, a.pose_update) <= 1e-9


def test_pcg_residual_property_at_scale(pv):
    """medium (1.25M observations): the returned update satisfies the reported relative
    residual when recomputed through the independently tested S'.v."""
    from paper_2405_05079_b200 import _lib, synth
    pr, _ = synth.make_problem("medium", 0)
    st = synth.random_state(pr, 1)
    dp = pv.DeviceProblem(pr, 0.1)
    sysm = pv.assemble_system(pr, st, 1, 1e-4, "pose_only", dp=dp)
    rep = pv.pcg_schur_solve(sysm, pv.SolverConfig(pcg_tolerance=1e-6, max_inner_iterations=300))
    assert rep.flag is None and rep.inner_iterations_used >= 1
    rhs = dp.debug(_lib.PV_DBG_RHS)[:, :12].ravel()
    U = dp.debug(_lib.PV_DBG_U).reshape(-1, 12, 12)
    x = rep.pose_update
    sx = np.einsum("nij,nj->ni", U, x.reshape(-1, 12)).ravel() - dp.schur_apply(1, x)
    got = np.linalg.norm(rhs - sx) / np.linalg.norm(rhs)
    # the recursive CG residual tracks the true one up to rounding
    assert abs(got - rep.truncation_estimate) <= 1e-3 * rep.truncation_estimate + 1e-10
    if rep.inner_iterations_used < 300:
        assert rep.truncation_estimate <= 1e-6

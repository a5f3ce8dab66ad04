"""GPU parity at BASELINE's larger configs and on the degenerate / error semantics.

Every expected value here comes from the REAL reference package
(tests/golden/make_golden_scale.py); the large problems are regenerated from the
seeded generator and pinned by a checksum.  Each test prints the achieved errors
(``pytest -s`` shows them; DESIGN.md section 2 records them).

* medium (356 cams / 226,730 landmarks / 1.25M obs), stage 1 from the N(0,1) start:
  first-iteration blocks and power solve per kernel (north_star: 1e-10 relative,
  norm-wise), then the 20-iteration lm_minimize trace (1e-6, same accept/reject
  string, same power orders).
* medium stage 2 (RiPoBA) from the lifted reference stage-1 result, TEACHER-FORCED
  (SURVEY App. B.3): at step k the device linearizes at the reference's state_k with
  the reference's lambda_k; its pose step, power order, landmark step and trial cost
  are compared; state_{k+1} is rebuilt from the reference's pose step through the
  device back-substitution (normal_eq.py:239-250).  The free-running 20-iteration
  trace is compared as far as it is not chaotic and the divergence point reported.
* large (5%, clustered visibility) and vlarge (1%, tracks up to 479) landmark
  subsamples: 10 stage-1 iterations (costs, accept string, power orders).
* degenerate landmark blocks (normal_eq.py:145-153,246-249; construction of
  pkg/tests/test_normal_eq.py:230-239 on a graph) and the stage-2 unit-norm
  ValueError (riemannian.py:46-48).
"""

import math

import numpy as np
import pytest

from _pvutil import check, golden, problem_from, rel

pytestmark = pytest.mark.gpu

TOL = 1e-10


@pytest.fixture(scope="module")
def pv():
    import paper_2405_05079_b200 as pv
    return pv


def _accept_string(costs):
    return "".join("A" if b < a else "R" for a, b in zip(costs, costs[1:]))


def _check_problem(problem, state, ck):
    assert problem.num_observations == int(ck[0])
    for got, want in ((problem.measurements.sum(), ck[1]), (problem.camera_indices.sum(), ck[2]),
                      (problem.landmark_indices.sum(), ck[3]), (state.cameras.sum(), ck[4]),
                      (state.landmarks.sum(), ck[5])):
        assert abs(float(got) - float(want)) <= 1e-9 * max(1.0, abs(float(want)))


def _sym6(a):
    return np.stack([a[:, 0, 0], a[:, 0, 1], a[:, 0, 2], a[:, 1, 1], a[:, 1, 2], a[:, 2, 2]], 1)


def _probes(n, seed=9):
    return np.random.Generator(np.random.Philox(seed)).standard_normal((4, n))


# --------------------------------------------------------------------------- medium, stage 1

@pytest.fixture(scope="module")
def medium(pv):
    from paper_2405_05079_b200 import synth
    z = golden("medium_s1.npz")
    problem, _ = synth.make_problem("medium", 0)
    state = synth.random_state(problem, 1)
    _check_problem(problem, state, z["checksum"])
    dp = pv.DeviceProblem(problem, 0.1)
    assert dp.n_l_local == problem.num_landmarks  # every landmark observed: local = global ids
    return z, problem, state, dp


def test_medium_first_iteration_per_kernel(pv, medium):
    from paper_2405_05079_b200 import _lib
    z, problem, state, dp = medium
    sysm = pv.assemble_system(problem, state, 1, 1e-4, "pose_only", dp=dp)
    n_p, sub = dp.n_p, z["subset"]
    err = {}
    err["U"] = rel(dp.debug(_lib.PV_DBG_U).reshape(n_p, 12, 12), z["U"])
    err["b_p"] = rel(dp.debug(_lib.PV_DBG_BP), z["b_p"])
    err["V"] = rel(dp.debug(_lib.PV_DBG_V)[sub], _sym6(z["V_sub"]))
    err["V+"] = rel(dp.debug(_lib.PV_DBG_VPINV)[sub], _sym6(z["Vp_sub"]))
    err["b_l"] = rel(dp.debug(_lib.PV_DBG_BL)[sub], z["b_l_sub"])
    assert int(dp.debug(_lib.PV_DBG_DEGEN).sum()) == int(z["n_degen"])
    err["S'v"] = rel(dp.schur_apply(1, z["probe"]), z["coupling"])
    rep = pv.power_schur_solve(sysm, pv.SolverConfig(max_power_order=20))
    err["rhs"] = rel(dp.debug(_lib.PV_DBG_RHS).ravel(), z["rhs"])
    assert rep.power_order_used == int(z["it1_order"])
    err["trunc"] = abs(rep.truncation_estimate - float(z["it1_trunc"])) / float(z["it1_trunc"])
    err["dx"] = rel(rep.pose_update, z["it1_dx"])
    dl = rep.landmark_update.reshape(-1, 3)
    err["dl(subset)"] = rel(dl[sub], z["it1_dl_sub"])
    err["|dl|"] = abs(np.linalg.norm(dl) - float(z["it1_dl_norm"])) / float(z["it1_dl_norm"])
    err["dl.probes"] = rel(_probes(dl.size) @ dl.ravel(), z["it1_dl_proj"])
    print("medium stage-1 first iteration, relative errors:",
          {k: f"{v:.1e}" for k, v in err.items()})
    for k, v in err.items():
        check("medium " + k, v, TOL)


def test_medium_stage1_trace(pv, medium):
    z, problem, state, dp = medium
    decisions = []
    _, trace = pv.lm_minimize(problem, state, 1, pv.SolverConfig(max_outer_iterations=20),
                              dp=dp, decisions=decisions)
    costs = np.array([r.cost for r in trace.records])
    ref = z["s1_costs"]
    worst = float(np.max(np.abs(costs[:len(ref)] - ref) / ref)) if len(costs) == len(ref) else 1
    print(f"medium stage-1 trace: {len(ref) - 1} iterations, max relative cost difference "
          f"{worst:.2e}, accept {_accept_string(ref)}")
    assert len(costs) == len(ref)
    np.testing.assert_allclose(costs, ref, rtol=1e-6, atol=0)
    assert _accept_string(costs) == _accept_string(ref)
    assert [d["order"] for d in decisions] == z["s1_orders"].tolist()


# --------------------------------------------------------------------------- medium, stage 2

@pytest.fixture(scope="module")
def medium2(pv, medium):
    _, problem, _, dp = medium
    z = golden("medium_s2.npz")
    start = pv.ProjectiveState(z["cams0"], z["lms0"])
    return z, problem, start, dp


def test_medium_stage2_teacher_forced(pv, medium2):
    z, problem, start, dp = medium2
    sub = z["subset"]
    dp.set_state(start)
    f0 = dp.cost(2)
    assert rel(f0, float(z["f0"])) <= 1e-12
    f = f0
    rows = []
    for k in range(len(z["tf_lam"])):
        lam = float(z["tf_lam"][k])
        dp.linearize(2)
        dp.damp(lam, True)
        order, trunc = dp.power_solve(20, 0.01)
        dx, dl = dp.step(2)
        dl = dl.reshape(-1, 3)
        e = dict(k=k, order=(order, int(z["tf_order"][k])),
                 dx=rel(dx, z["tf_dx"][k]),
                 trunc=abs(trunc - z["tf_trunc"][k]) / z["tf_trunc"][k],
                 dl_sub=rel(dl[sub], z["tf_dl_sub"][k]),
                 dl_norm=abs(np.linalg.norm(dl) - z["tf_dl_norm"][k]) / z["tf_dl_norm"][k],
                 dl_proj=rel(_probes(dl.size) @ dl.ravel(), z["tf_dl_proj"][k]))
        # own trial from the device's own step
        assert dp.trial(2)
        f_own = dp.cost(2, trial=True)
        # teacher forcing: the reference's pose step, back-substituted on the device
        dp.back_substitute(z["tf_dx"][k])
        assert dp.trial(2)
        f_trial = dp.cost(2, trial=True)
        e["f_trial(own step)"] = rel(f_own, z["tf_f_trial"][k])
        e["f_trial(ref step)"] = rel(f_trial, z["tf_f_trial"][k])
        acc = f_trial < f
        assert acc == bool(z["tf_accepted"][k])
        assert (f_own < f) == acc
        rows.append(e)
        if acc:
            dp.accept(2, resolve=False)
            f = f_trial
    for e in rows:
        print("medium stage-2 teacher-forced step", e["k"], "order", e["order"],
              {k: f"{v:.1e}" for k, v in e.items() if k not in ("k", "order")},
              "reference's own 1e-16 floor:",
              {q: f"{z['floor_' + q][e['k']]:.1e}" for q in ("dx", "dl_proj", "f_trial", "trunc")})
    # This chain starts from an unconverged stage-1 result (stage-2 cost 2.3e9) and is
    # ill-conditioned: the REFERENCE moves its own dx by up to ~7e-7 and f_trial by up to
    # ~2e-2 when state_k is perturbed by 1e-16 (floor_*, make_golden_scale.py).  Asserted:
    # every decision (power order, accept/reject: above); the step within 10x the
    # reference's own floor (max over three perturbations); and the teacher-forced trial
    # cost -- the reference's dx, device back-substitution and cost -- within north_star's
    # 1e-6.  The trial cost of the device's OWN step is reported, not asserted: it is
    # hypersensitive to the step (observations with |z| near 0 dominate this cost), e.g.
    # at step 4 a 1.7e-8 relative change of dx moves it by ~2e-4.
    for e in rows:
        k = e["k"]
        assert e["order"][0] == e["order"][1]
        for q, fq in (("dx", "dx"), ("dl_proj", "dl_proj"), ("trunc", "trunc")):
            check(f"medium s2 step {k} {q} (floor {z['floor_' + fq][k]:.1e})", e[q],
                  max(10 * float(z["floor_" + fq][k]), 1e-10))
        check(f"medium s2 step {k} f_trial(ref step)", e["f_trial(ref step)"], 1e-6)


def test_medium_stage2_free_running(pv, medium2):
    """Free-running RiPoBA from the identical lifted start.  Stage 2 is chaotic along
    near-flat directions: the trace must agree within 1e-6 while the
    runs have not diverged; the divergence iteration is reported, not asserted."""
    z, problem, start, dp = medium2
    decisions = []
    _, trace = pv.lm_minimize(problem, start, 2, pv.SolverConfig(max_outer_iterations=20),
                              dp=dp, decisions=decisions)
    costs = np.array([r.cost for r in trace.records])
    ref = z["s2_costs"]
    n = min(len(costs), len(ref))
    d = np.abs(costs[:n] - ref[:n]) / ref[:n]
    div = next((i for i in range(n) if d[i] > 1e-6), None)
    pert = z["s2_costs_perturbed"]
    m = min(len(pert), len(ref))
    dp_ = np.abs(pert[:m] - ref[:m]) / ref[:m]
    div_ref = next((i for i in range(m) if dp_[i] > 1e-6), None)
    print(f"medium stage-2 free-running: {n - 1} iterations compared, max relative cost "
          f"difference {d.max():.2e}, first > 1e-6 at iteration {div}; the reference from a "
          f"1e-16-perturbed start first differs > 1e-6 at iteration {div_ref}; accept ours "
          f"{_accept_string(costs)} ref {_accept_string(ref)}")
    # identical up to the first accepted step, whose trial cost is chaotic (see the
    # teacher-forced test); the rest is the divergence report above
    np.testing.assert_allclose(costs[:3], ref[:3], rtol=1e-6, atol=0)
    assert _accept_string(costs[:4]) == _accept_string(ref[:4])
    assert [x["order"] for x in decisions[:3]] == z["s2_orders"][:3].tolist()


# --------------------------------------------------------------------------- medium, stage 2 GT

def test_medium_stage2_refinement_per_kernel(pv, medium):
    """Stage 2 as a refinement from the lifted noisy ground truth (well conditioned: the
    reference's own dx moves by ~1e-13 under a 1e-16 perturbation): per-kernel parity at
    north_star's 1e-10 and the free-running trace."""
    from paper_2405_05079_b200 import _lib
    _, problem, _, dp = medium
    z = golden("medium_s2gt.npz")
    st = pv.ProjectiveState(z["cams0"], z["lms0"])
    sub = z["subset"]
    sysm = pv.assemble_system(problem, st, 2, 1e-4, "both", dp=dp)
    n_p = dp.n_p
    err = {"f0": rel(dp.cost(2), float(z["f0"]))}
    err["U"] = rel(dp.debug(_lib.PV_DBG_U).reshape(n_p, 12, 12)[:, :11, :11], z["U"])
    err["b_p"] = rel(dp.debug(_lib.PV_DBG_BP)[:, :11], z["b_p"])
    err["V+"] = rel(dp.debug(_lib.PV_DBG_VPINV)[sub], _sym6(z["Vp_sub"]))
    err["b_l"] = rel(dp.debug(_lib.PV_DBG_BL)[sub], z["b_l_sub"])
    assert int(dp.debug(_lib.PV_DBG_DEGEN).sum()) == int(z["n_degen"])
    err["S'v"] = rel(dp.schur_apply(2, z["probe"]), z["coupling"])
    rep = pv.power_schur_solve(sysm, pv.SolverConfig(max_power_order=20))
    err["rhs"] = rel(dp.debug(_lib.PV_DBG_RHS)[:, :11].ravel(), z["rhs"])
    assert rep.power_order_used == int(z["it1_order"])
    err["trunc"] = abs(rep.truncation_estimate - float(z["it1_trunc"])) / float(z["it1_trunc"])
    err["dx"] = rel(rep.pose_update, z["it1_dx"])
    dl = rep.landmark_update.reshape(-1, 3)
    err["dl(subset)"] = rel(dl[sub], z["it1_dl_sub"])
    err["dl.probes"] = rel(_probes(dl.size) @ dl.ravel(), z["it1_dl_proj"])
    assert dp.trial(2)
    err["f_trial"] = rel(dp.cost(2, trial=True), float(z["it1_f_trial"]))
    print("medium stage-2 refinement first iteration, relative errors:",
          {k: f"{v:.1e}" for k, v in err.items()}, f"(reference floor dx {float(z['floor_dx']):.1e})")
    for k, v in err.items():
        check("medium s2 refinement " + k, v, TOL)
    decisions = []
    _, trace = pv.lm_minimize(problem, st, 2, pv.SolverConfig(max_outer_iterations=20), dp=dp,
                              decisions=decisions)
    costs = np.array([r.cost for r in trace.records])
    ref = z["s2_costs"]
    assert len(costs) == len(ref)
    print(f"medium stage-2 refinement trace: max relative cost difference "
          f"{np.max(np.abs(costs - ref) / ref):.2e}")
    np.testing.assert_allclose(costs, ref, rtol=1e-6, atol=0)
    assert _accept_string(costs) == _accept_string(ref)
    assert [x["order"] for x in decisions] == z["s2_orders"].tolist()


# --------------------------------------------------------------------------- subsamples

@pytest.mark.parametrize("name", ["large", "vlarge"])
def test_subsample_stage1_traces(pv, name):
    from paper_2405_05079_b200 import synth
    z = golden("subsample_lm.npz")
    problem, _ = synth.make_problem(name, 0, landmark_fraction=float(z[name + "_fraction"]))
    state = synth.random_state(problem, 1)
    _check_problem(problem, state, z[name + "_checksum"])
    decisions = []
    cfg = pv.SolverConfig(max_outer_iterations=10, max_power_order=int(z[name + "_max_order"]))
    _, trace = pv.lm_minimize(problem, state, 1, cfg, decisions=decisions)
    costs = np.array([r.cost for r in trace.records])
    ref = z[name + "_costs"]
    worst = float(np.max(np.abs(costs - ref) / ref)) if len(costs) == len(ref) else math.inf
    print(f"{name} subsample ({problem.num_observations} obs, max track "
          f"{np.bincount(problem.landmark_indices).max()}): max relative cost difference "
          f"{worst:.2e}, accept {_accept_string(ref)}")
    assert len(costs) == len(ref)
    np.testing.assert_allclose(costs, ref, rtol=1e-6, atol=0)
    assert _accept_string(costs) == _accept_string(ref)
    assert [d["order"] for d in decisions] == z[name + "_orders"].tolist()


# --------------------------------------------------------------------------- degenerate blocks

@pytest.fixture(scope="module")
def degen():
    return golden("degen.npz")


@pytest.mark.parametrize("tag,mode", [("v_", "pose_only"), ("j_", "both")])
def test_degenerate_landmark_blocks(pv, degen, tag, mode):
    from paper_2405_05079_b200 import _lib
    z = degen
    problem = problem_from(z)
    dp = pv.DeviceProblem(problem, 0.1)
    st = pv.ProjectiveState(z["cams"], z["lms"])
    sysm = pv.assemble_system(problem, st, 1, float(z[tag + "lam"]), mode, dp=dp)
    flags = dp.debug(_lib.PV_DBG_DEGEN) != 0
    np.testing.assert_array_equal(flags, z[tag + "degen"])
    assert sysm.n_degenerate == int(z[tag + "degen"].sum())
    err = {"V+": rel(dp.debug(_lib.PV_DBG_VPINV), _sym6(z[tag + "Vp"]))}
    if mode == "pose_only":
        err["V"] = rel(dp.debug(_lib.PV_DBG_V), _sym6(z[tag + "V"]))
    rep = pv.power_schur_solve(sysm, pv.SolverConfig(max_power_order=20))
    err["rhs"] = rel(dp.debug(_lib.PV_DBG_RHS).ravel(), z[tag + "rhs"])
    assert rep.power_order_used == int(z[tag + "order"])
    err["dx"] = rel(rep.pose_update, z[tag + "dx"])
    err["dl"] = rel(rep.landmark_update, z[tag + "dl"])
    dl = rep.landmark_update.reshape(-1, 3)
    assert not dl[z[tag + "degen"]].any()  # exactly zero (normal_eq.py:246-247)
    back = pv.back_substitute(sysm, np.ones(sysm.pose_dim))
    err["backsub(1)"] = rel(back, z[tag + "backsub_ones"])
    assert not back.reshape(-1, 3)[z[tag + "degen"]].any()
    print(f"degenerate blocks ({mode}): {int(flags.sum())} flagged, relative errors",
          {k: f"{v:.1e}" for k, v in err.items()})
    for k, v in err.items():
        check(f"degen {mode} {k}", v, TOL)


def test_degenerate_graph_resolve_and_trace(pv, degen):
    z = degen
    problem = problem_from(z)
    dp = pv.DeviceProblem(problem, 0.1)
    st = pv.ProjectiveState(z["cams"], z["lms"])
    assert rel(pv.total_cost(st, problem, 1, dp=dp), z["cost_s1"]) <= 1e-13
    out = pv.solve_landmarks(st, problem, dp=dp)
    assert rel(out, z["resolved"]) <= TOL
    _, trace = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=6), dp=dp)
    costs = np.array([r.cost for r in trace.records])
    np.testing.assert_allclose(costs, z["lm_costs"], rtol=1e-6, atol=0)
    assert _accept_string(costs) == _accept_string(z["lm_costs"])


def test_stage2_non_unit_state_raises(pv, degen):
    """riemannian.py:46-48 through lm_minimize (after the initial trace record, as the
    reference) and riemannian_step."""
    z = degen
    problem = problem_from(z)
    st = pv.ProjectiveState(z["cams"], z["lms"])
    seen = []
    with pytest.raises(ValueError) as ei:
        pv.lm_minimize(problem, st, 2, pv.SolverConfig(max_outer_iterations=2),
                       trace_sink=seen.append)
    assert str(ei.value) == str(z["nonunit_message"])
    assert len(seen) == 1 and seen[0].iteration == 0
    with pytest.raises(ValueError):
        pv.riemannian_step(problem, st, pv.SolverConfig())

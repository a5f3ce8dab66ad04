"""Scale and edge-case golden fixtures from the REAL reference package (build container only).

Run from the repo root:
    python tests/golden/make_golden_scale.py [medium|floor|gt|subsample|degen|all]

Like make_golden.py it imports ``stratba`` read-only from /root/reference/pkg/src and
stores the reference's own outputs.  The large problems themselves are NOT stored: the
GPU tests regenerate them with the seeded generator (paper_2405_05079_b200/synth.py,
Philox: bit-identical on every machine) and a checksum in each fixture pins that.

medium_s1.npz -- BASELINE medium config (356 cams / 226,730 landmarks / 1.25M obs),
    seed 0, N(0,1) start (seed 1):
    * the first LM iteration's blocks (solvers.py:351-353): damped U, b_p, schur_rhs,
      the coupling round trip S'.v of a probe (solvers.py:117-123), the power solve
      (dx, order, truncation) and, for a deterministic subset of landmarks
      (every 97th), V, V+, b_l and the back-substituted update;
    * the stage-1 lm_minimize trace (20 iterations) with the power order of every
      inner solve.
medium_s2.npz -- stage 2 (RiPoBA) from the lifted reference stage-1 result:
    * the lifted start state (the one stored array of problem size);
    * TEACHER-FORCED steps: at step k the reference's (state_k,
      lambda_k) -> riemannian_step -> apply_tangent_step -> total_cost; stored are
      lambda_k, dx_k, the power order / truncation, checksums and a landmark subset
      of dl_k, f_trial_k and the accept decision.  The GPU test rebuilds state_{k+1}
      from the reference's dx_k (back_substitute, normal_eq.py:239-250), so both sides
      linearize at the same point every step;
    * the free-running 20-iteration stage-2 lm_minimize trace (divergence report).
    * the reference's own conditioning floor on that chain ("floor"): the spread of its dx,
      dl and f_trial when state_k is perturbed by 1e-16 relative, and its free-running
      trace from a 1e-16-perturbed start.
medium_s2gt.npz -- stage 2 as a refinement from the lifted, noisy ground truth (a
    well-conditioned chain): first-iteration per-kernel quantities, the reference's
    own 1e-16 sensitivity, and the 20-iteration free-running trace.
subsample_lm.npz -- landmark subsamples of the large (5%, clustered visibility) and
    vlarge (1%, power-law tracks up to 500) configs: 10 stage-1 iterations each, costs
    and power orders.
degen.npz -- degenerate landmark blocks (normal_eq.py:145-153,246-249; the construction
    of pkg/tests/test_normal_eq.py:230-239 on a whole graph): cameras whose first three
    columns vanish (J_l = 0) or whose third column vanishes (rank-2 J_l).  assemble in
    both damping modes, V+, degenerate flags, power solve + back-substitution, the
    landmark re-solve (rank-deficient landmarks untouched) and a 6-iteration LM trace;
    plus the stage-2 non-unit-state ValueError message (riemannian.py:46-48).
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, REF)
sys.path.insert(0, str(ROOT))

import stratba  # noqa: E402
from stratba import normal_eq, objective, riemannian, solvers  # noqa: E402

from paper_2405_05079_b200 import synth  # noqa: E402

SUBSET_STRIDE = 97


def ref_problem(p):
    return stratba.BaProblem(p.num_cameras, p.num_landmarks, p.num_observations,
                             p.camera_indices, p.landmark_indices, p.measurements)


def checksum(problem, state):
    return np.array([problem.num_observations, float(problem.measurements.sum()),
                     float(problem.camera_indices.sum()), float(problem.landmark_indices.sum()),
                     float(state.cameras.sum()), float(state.landmarks.sum())])


class OrderLog:
    """Records (order, truncation) of every power solve without changing it."""

    def __init__(self):
        self.orders, self.truncs = [], []
        self._orig = solvers._INNER_SOLVERS["power"]

    def __enter__(self):
        def wrapped(system, config):
            rep = self._orig(system, config)
            self.orders.append(rep.power_order_used)
            self.truncs.append(rep.truncation_estimate)
            return rep
        solvers._INNER_SOLVERS["power"] = wrapped
        return self

    def __exit__(self, *a):
        solvers._INNER_SOLVERS["power"] = self._orig


def probe_vectors(n, seed):
    rng = np.random.Generator(np.random.Philox(seed))
    return rng.standard_normal((4, n))


def make_medium():
    pose = objective.PoseConfig(0.1)
    problem, _ = synth.make_problem("medium", 0)
    state = synth.random_state(problem, 1)
    rp = ref_problem(problem)
    st = stratba.ProjectiveState(state.cameras, state.landmarks)
    out = {"checksum": checksum(problem, state)}
    subset = np.arange(0, problem.num_landmarks, SUBSET_STRIDE)
    out["subset"] = subset
    cfg = solvers.SolverConfig(max_outer_iterations=20, max_power_order=20)
    # first LM iteration, per-kernel quantities
    t = time.time()
    system = normal_eq.assemble(normal_eq.build_stage1_blocks(rp, st, pose), cfg.initial_lambda,
                                normal_eq.POSE_ONLY)
    out["U"], out["b_p"] = system.u_blocks, system.b_p
    out["rhs"] = normal_eq.schur_rhs(system)
    probe = np.random.Generator(np.random.Philox(5)).standard_normal(system.pose_dim)
    out["probe"] = probe
    out["coupling"] = solvers._coupling_round_trip(system, probe)
    out["n_degen"] = int(system.v_degenerate.sum())
    out["V_sub"], out["Vp_sub"] = system.v_blocks[subset], system.v_inv[subset]
    out["b_l_sub"] = system.b_l[subset]
    rep = solvers.power_schur_solve(system, cfg)
    out["it1_dx"], out["it1_order"] = rep.pose_update, rep.power_order_used
    out["it1_trunc"] = rep.truncation_estimate
    dl = rep.landmark_update.reshape(-1, 3)
    out["it1_dl_sub"] = dl[subset]
    out["it1_dl_norm"] = float(np.linalg.norm(dl))
    out["it1_dl_proj"] = probe_vectors(dl.size, 9) @ dl.ravel()
    print("medium first iteration", time.time() - t, "order", rep.power_order_used)
    del system
    t = time.time()
    with OrderLog() as log:
        s1, tr = solvers.lm_minimize(rp, st, 1, cfg)
    out["s1_costs"] = np.array([r.cost for r in tr.records])
    out["s1_orders"] = np.array(log.orders)
    print("medium stage 1", time.time() - t, out["s1_costs"][-1], log.orders)
    np.savez_compressed(OUT / "medium_s1.npz", **out)

    # ---- stage 2 from the lifted reference result
    lifted = riemannian.lift_stage1_to_stage2(s1)
    out2 = {"checksum": checksum(problem, state), "subset": subset,
            "cams0": lifted.cameras, "lms0": lifted.landmarks}
    cfg2 = solvers.SolverConfig(max_outer_iterations=20, max_power_order=20)
    st_k = lifted
    f = objective.total_cost(st_k, rp, 2)
    lam = cfg2.initial_lambda
    out2["f0"] = f
    rec = {k: [] for k in ("lam", "dx", "order", "trunc", "dl_sub", "dl_norm", "dl_proj",
                           "f_trial", "accepted")}
    t = time.time()
    for k in range(5):
        bases = riemannian.state_tangent_bases(st_k)
        rep = riemannian.riemannian_step(rp, st_k, cfg2, lam, bases)
        trial = riemannian.apply_tangent_step(st_k, bases, rep)
        f_trial = objective.total_cost(trial, rp, 2) if trial is not None else np.inf
        dl = rep.landmark_update.reshape(-1, 3)
        rec["lam"].append(lam)
        rec["dx"].append(rep.pose_update)
        rec["order"].append(rep.power_order_used)
        rec["trunc"].append(rep.truncation_estimate)
        rec["dl_sub"].append(dl[subset])
        rec["dl_norm"].append(float(np.linalg.norm(dl)))
        rec["dl_proj"].append(probe_vectors(dl.size, 9) @ dl.ravel())
        rec["f_trial"].append(f_trial)
        acc = f_trial < f
        rec["accepted"].append(acc)
        if acc:
            st_k, f = trial, f_trial
            lam = max(cfg2.lambda_min, lam * cfg2.lambda_decrease)
        else:
            lam = min(cfg2.lambda_max, lam * cfg2.lambda_increase)
        print("medium stage 2 step", k, f_trial, acc, rep.power_order_used, time.time() - t)
    for k, v in rec.items():
        out2["tf_" + k] = np.array(v)
    t = time.time()
    with OrderLog() as log:
        _, tr2 = solvers.lm_minimize(rp, lifted, 2, cfg2)
    out2["s2_costs"] = np.array([r.cost for r in tr2.records])
    out2["s2_orders"] = np.array(log.orders)
    print("medium stage 2 free", time.time() - t, out2["s2_costs"])
    # the free-running trace and the teacher-forced decisions are the same computation
    # for the first steps (identical inputs): a self-check of this script
    fr = out2["s2_costs"]
    acc_fr = fr[1:6] < fr[:5]
    assert np.array_equal(acc_fr[:len(rec["accepted"])], np.array(rec["accepted"])), (acc_fr,
                                                                                      rec)
    np.savez_compressed(OUT / "medium_s2.npz", **out2)


def make_subsample():
    out = {}
    for name, frac, max_order in (("large", 0.05, 20), ("vlarge", 0.01, 30)):
        problem, _ = synth.make_problem(name, 0, landmark_fraction=frac)
        state = synth.random_state(problem, 1)
        rp = ref_problem(problem)
        st = stratba.ProjectiveState(state.cameras, state.landmarks)
        cfg = solvers.SolverConfig(max_outer_iterations=10, max_power_order=max_order)
        t = time.time()
        with OrderLog() as log:
            _, tr = solvers.lm_minimize(rp, st, 1, cfg)
        out[name + "_checksum"] = checksum(problem, state)
        out[name + "_fraction"] = frac
        out[name + "_max_order"] = max_order
        out[name + "_costs"] = np.array([r.cost for r in tr.records])
        out[name + "_orders"] = np.array(log.orders)
        k = np.bincount(problem.landmark_indices)
        print(name, frac, problem.num_observations, "max k", k.max(), time.time() - t,
              out[name + "_costs"][[0, -1]], log.orders)
    np.savez_compressed(OUT / "subsample_lm.npz", **out)


def degenerate_graph():
    """6 cameras, 60 landmarks.  Cameras 0-1 get a zero third column (rank-2 J_l for the
    landmarks only they observe), camera 2 a zero left 3x3 block (J_l = 0)."""
    rng = np.random.default_rng(31)
    n_p, n_l = 6, 60
    ci, li = [], []
    for j in range(n_l):
        if j < 6:          # seen only by cameras 0 and 1
            cams = [0, 1]
        elif j < 9:        # seen only by camera 2 (twice is not allowed: one camera)
            cams = [2]
        elif j < 12:       # cameras 0 and 2: rank-2 rows plus zero rows
            cams = [0, 2]
        else:
            cams = sorted(rng.choice(n_p, size=int(rng.integers(2, 5)), replace=False).tolist())
        for c in cams:
            ci.append(c)
            li.append(j)
    perm = rng.permutation(len(ci))
    meas = rng.standard_normal((len(ci), 2))
    problem = stratba.BaProblem(n_p, n_l, len(ci), np.array(ci)[perm], np.array(li)[perm], meas)
    cams = rng.standard_normal((n_p, 3, 4))
    cams[0:2, :, 2] = 0.0
    cams[2, :, :3] = 0.0
    lms = np.concatenate([rng.standard_normal((n_l, 3)), np.ones((n_l, 1))], axis=1)
    return problem, stratba.ProjectiveState(cams, lms)


def make_degen():
    pose = objective.PoseConfig(0.1)
    problem, st = degenerate_graph()
    out = dict(n_cameras=problem.num_cameras, n_landmarks=problem.num_landmarks,
               cam_idx=problem.camera_indices, lm_idx=problem.landmark_indices,
               meas=problem.measurements, cams=st.cameras, lms=st.landmarks)
    cfg = solvers.SolverConfig(max_power_order=20, power_threshold=0.01)
    blocks = normal_eq.build_stage1_blocks(problem, st, pose)
    for lam, mode, tag in ((1e-4, normal_eq.POSE_ONLY, "v_"), (0.3, normal_eq.BOTH, "j_")):
        system = normal_eq.assemble(blocks, lam, mode)
        out[tag + "lam"] = lam
        out[tag + "V"], out[tag + "Vp"] = system.v_blocks, system.v_inv
        out[tag + "degen"] = system.v_degenerate
        out[tag + "rhs"] = normal_eq.schur_rhs(system)
        rep = solvers.power_schur_solve(system, cfg)
        out[tag + "dx"], out[tag + "dl"] = rep.pose_update, rep.landmark_update
        out[tag + "order"] = rep.power_order_used
        ones = np.ones(system.pose_dim)
        out[tag + "backsub_ones"] = normal_eq.back_substitute(system, ones)
        print("degen", tag, "degenerate", np.nonzero(system.v_degenerate)[0])
    out["resolved"] = objective.solve_landmarks(st, problem, pose)
    out["cost_s1"] = objective.total_cost(st, problem, 1, pose)
    _, tr = solvers.lm_minimize(problem, st, 1, solvers.SolverConfig(max_outer_iterations=6))
    out["lm_costs"] = np.array([r.cost for r in tr.records])
    # stage 2 on a state that is not on the unit spheres: ValueError before any step
    try:
        solvers.lm_minimize(problem, st, 2, solvers.SolverConfig(max_outer_iterations=2))
        raise AssertionError("expected ValueError")
    except ValueError as exc:
        out["nonunit_message"] = str(exc)
    print("degen lm", out["lm_costs"], out["nonunit_message"])
    np.savez_compressed(OUT / "degen.npz", **out)


def _perturbed(state, eps, seed):
    """The state with every coordinate scaled by (1 + eps N(0,1)), retracted."""
    rng = np.random.default_rng(seed)
    c = state.cameras * (1 + eps * rng.standard_normal(state.cameras.shape))
    lm = state.landmarks * (1 + eps * rng.standard_normal(state.landmarks.shape))
    return riemannian.retract(stratba.ProjectiveState(c, lm))


def make_medium_floor():
    """The reference's OWN sensitivity on the medium stage-2 chain (added to medium_s2.npz).

    For each teacher-forced step k the reference re-runs riemannian_step + trial cost
    from its state_k perturbed by 1e-16 relative (three seeds): the spread of dx, dl and
    f_trial is the conditioning floor no implementation can beat.  The free-running
    trace is re-run from a perturbed start as well (the reference's own divergence)."""
    z = dict(np.load(OUT / "medium_s2.npz"))
    problem, _ = synth.make_problem("medium", 0)
    rp = ref_problem(problem)
    cfg2 = solvers.SolverConfig(max_outer_iterations=20, max_power_order=20)
    st_k = stratba.ProjectiveState(z["cams0"], z["lms0"])
    floor = {"dx": [], "dl_proj": [], "f_trial": [], "trunc": []}
    t = time.time()
    for k in range(len(z["tf_lam"])):
        lam = float(z["tf_lam"][k])
        worst = dict.fromkeys(floor, 0.0)
        for seed in range(3):
            sp = _perturbed(st_k, 1e-16, 100 + seed)
            bases = riemannian.state_tangent_bases(sp)
            rep = riemannian.riemannian_step(rp, sp, cfg2, lam, bases)
            trial = riemannian.apply_tangent_step(sp, bases, rep)
            f_tr = objective.total_cost(trial, rp, 2)
            dl = rep.landmark_update
            proj = probe_vectors(dl.size, 9) @ dl
            worst["dx"] = max(worst["dx"], np.linalg.norm(rep.pose_update - z["tf_dx"][k])
                              / np.linalg.norm(z["tf_dx"][k]))
            worst["dl_proj"] = max(worst["dl_proj"], np.linalg.norm(proj - z["tf_dl_proj"][k])
                                   / np.linalg.norm(z["tf_dl_proj"][k]))
            worst["f_trial"] = max(worst["f_trial"],
                                   abs(f_tr - z["tf_f_trial"][k]) / z["tf_f_trial"][k])
            worst["trunc"] = max(worst["trunc"], abs(rep.truncation_estimate - z["tf_trunc"][k])
                                 / z["tf_trunc"][k])
        for q in floor:
            floor[q].append(worst[q])
        print("floor step", k, {q: f"{v:.1e}" for q, v in worst.items()}, time.time() - t,
              flush=True)
        # the reference's own next state (its step from the unperturbed state_k)
        bases = riemannian.state_tangent_bases(st_k)
        if bool(z["tf_accepted"][k]):
            rep = riemannian.riemannian_step(rp, st_k, cfg2, lam, bases)
            st_k = riemannian.apply_tangent_step(st_k, bases, rep)
    for q, v in floor.items():
        z["floor_" + q] = np.array(v)
    _, tr = solvers.lm_minimize(rp, _perturbed(stratba.ProjectiveState(z["cams0"], z["lms0"]),
                                               1e-16, 7), 2, cfg2)
    z["s2_costs_perturbed"] = np.array([r.cost for r in tr.records])
    print("perturbed free run", z["s2_costs_perturbed"])
    np.savez_compressed(OUT / "medium_s2.npz", **z)


def make_medium_gt():
    """medium_s2gt.npz -- stage 2 where RiPoBA is used as a refinement: from the lifted
    ground truth with noise (cameras x (1 + 1e-3 N), landmarks + 1e-2 N), a
    well-conditioned chain.  First-iteration per-kernel quantities, the reference's own
    1e-16 sensitivity of dx, and the 20-iteration free-running trace."""
    problem, truth = synth.make_problem("medium", 0)
    rp = ref_problem(problem)
    gt = synth.ground_truth_state(truth)
    rng = np.random.default_rng(11)
    cams = gt.cameras * (1 + 1e-3 * rng.standard_normal(gt.cameras.shape))
    lms = np.array(gt.landmarks)
    lms[:, :3] += 1e-2 * rng.standard_normal((len(lms), 3))
    st = riemannian.lift_stage1_to_stage2(stratba.ProjectiveState(cams, lms))
    out = {"checksum": checksum(problem, stratba.ProjectiveState(cams, lms)),
           "cams0": st.cameras, "lms0": st.landmarks}
    subset = np.arange(0, problem.num_landmarks, SUBSET_STRIDE)
    out["subset"] = subset
    cfg = solvers.SolverConfig(max_outer_iterations=20, max_power_order=20)
    lam = cfg.initial_lambda
    bases = riemannian.state_tangent_bases(st)
    system = normal_eq.assemble(riemannian.project_blocks(normal_eq.build_stage2_blocks(rp, st),
                                                          bases), lam, normal_eq.BOTH)
    out["f0"] = objective.total_cost(st, rp, 2)
    out["U"], out["b_p"] = system.u_blocks, system.b_p
    out["rhs"] = normal_eq.schur_rhs(system)
    probe = np.random.Generator(np.random.Philox(5)).standard_normal(system.pose_dim)
    out["probe"] = probe
    out["coupling"] = solvers._coupling_round_trip(system, probe)
    out["V_sub"], out["Vp_sub"] = system.v_blocks[subset], system.v_inv[subset]
    out["b_l_sub"] = system.b_l[subset]
    out["n_degen"] = int(system.v_degenerate.sum())
    rep = solvers.power_schur_solve(system, cfg)
    out["it1_dx"], out["it1_order"] = rep.pose_update, rep.power_order_used
    out["it1_trunc"] = rep.truncation_estimate
    dl = rep.landmark_update.reshape(-1, 3)
    out["it1_dl_sub"] = dl[subset]
    out["it1_dl_proj"] = probe_vectors(dl.size, 9) @ dl.ravel()
    trial = riemannian.apply_tangent_step(st, bases, rep)
    out["it1_f_trial"] = objective.total_cost(trial, rp, 2)
    fl = 0.0
    for seed in range(3):
        sp = _perturbed(st, 1e-16, 200 + seed)
        r2 = riemannian.riemannian_step(rp, sp, cfg, lam, riemannian.state_tangent_bases(sp))
        fl = max(fl, np.linalg.norm(r2.pose_update - rep.pose_update)
                 / np.linalg.norm(rep.pose_update))
    out["floor_dx"] = fl
    print("medium gt first step order", rep.power_order_used, "dx floor", fl, flush=True)
    t = time.time()
    with OrderLog() as log:
        _, tr = solvers.lm_minimize(rp, st, 2, cfg)
    out["s2_costs"] = np.array([r.cost for r in tr.records])
    out["s2_orders"] = np.array(log.orders)
    print("medium gt stage 2", time.time() - t, out["s2_costs"], log.orders)
    np.savez_compressed(OUT / "medium_s2gt.npz", **out)


if __name__ == "__main__":
    print("numpy", np.__version__)
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("degen", "all"):
        make_degen()
    if what in ("subsample", "all"):
        make_subsample()
    if what in ("medium", "all"):
        make_medium()
    if what in ("floor", "medium", "all"):
        make_medium_floor()
    if what in ("gt", "all"):
        make_medium_gt()

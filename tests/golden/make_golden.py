"""Generate golden fixtures from the REAL reference package (build container only).

Run from the repo root:  python tests/golden/make_golden.py
It imports ``stratba`` read-only from /root/reference/pkg/src, runs the
reference's own functions on seeded inputs, and stores inputs + outputs as
compressed .npz fixtures in tests/golden/.  /root/reference does not exist on
the GPU box; the fixtures travel instead.

Fixtures
--------
mini_s1.npz / mini_s2.npz  -- small random graphs (reference conftest style):
    assemble() blocks mapped to landmark-CSR order, schur_rhs, S'.v of a probe
    vector, power_schur_solve (threshold 0.01 and 0), back-substitution,
    solve_landmarks, total_cost; stage 2 uses project_blocks + BOTH damping.
tiny_lm.npz  -- BASELINE tiny config: reference stage-1 lm_minimize (20 its),
    first-iteration power solve, stage-2 lm_minimize from the lifted result
    (12 its) and its first riemannian_step.
small_lm.npz -- BASELINE small config: reference stage-1 cost trace (50 its).
pcg.npz      -- the PCG inner solver (solvers.py:153-187) on the mini graphs:
    schur_diag_blocks and pcg_schur_solve at three (tolerance, cap) settings for
    the stage-1 varpro / joint and stage-2 systems, plus lm_minimize traces with
    inner_solver="pcg" (stage 1 and 2) on the mini graphs and the tiny config.

``python tests/golden/make_golden.py pcg`` regenerates pcg.npz only.
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


def csr_positions(problem):
    order, ids, counts = objective.landmark_order(problem)
    offsets = np.zeros(problem.num_landmarks + 1, dtype=np.int64)
    full_counts = np.zeros(problem.num_landmarks, dtype=np.int64)
    full_counts[ids] = counts
    np.cumsum(full_counts, out=offsets[1:])
    return offsets


def blocks_to_csr(problem, system):
    offsets = csr_positions(problem)
    d_p, d_l = system.pose_width, system.lm_width
    W = np.zeros((problem.num_observations, d_p, d_l))
    for g, w in zip(system.groups, system.w_blocks):
        k = g.cams.shape[1]
        pos = offsets[g.lm_ids][:, None] + np.arange(k)[None, :]
        W[pos.ravel()] = w.reshape(-1, d_p, d_l)
    return W


def random_graph(n_cameras, n_landmarks, seed):
    rng = np.random.default_rng(seed)
    ci, li = [], []
    for j in range(n_landmarks):
        k = int(rng.integers(2, n_cameras + 1))
        for c in sorted(rng.choice(n_cameras, size=k, replace=False)):
            ci.append(c)
            li.append(j)
    # shuffle the observation order so CSR sorting is exercised
    perm = rng.permutation(len(ci))
    meas = 2.0 * rng.standard_normal((len(ci), 2))
    return stratba.BaProblem(n_cameras, n_landmarks, len(ci), np.array(ci)[perm],
                             np.array(li)[perm], meas)


def problem_arrays(p):
    return dict(n_cameras=p.num_cameras, n_landmarks=p.num_landmarks,
                cam_idx=p.camera_indices.astype(np.int32),
                lm_idx=p.landmark_indices.astype(np.int32), meas=p.measurements)


def system_arrays(prefix, problem, system, cfg_thr, cfg_zero, probe):
    out = {}
    out[prefix + "U"] = system.u_blocks
    out[prefix + "V"] = system.v_blocks
    out[prefix + "Vp"] = system.v_inv
    out[prefix + "degen"] = system.v_degenerate
    out[prefix + "W"] = blocks_to_csr(problem, system)
    out[prefix + "b_p"] = system.b_p
    out[prefix + "b_l"] = system.b_l
    out[prefix + "rhs"] = normal_eq.schur_rhs(system)
    out[prefix + "coupling"] = solvers._coupling_round_trip(system, probe)
    out[prefix + "apply_schur"] = normal_eq.apply_schur(system, probe)
    for tag, cfg in (("thr", cfg_thr), ("zero", cfg_zero)):
        rep = solvers.power_schur_solve(system, cfg)
        out[prefix + f"pow_{tag}_dx"] = rep.pose_update
        out[prefix + f"pow_{tag}_dl"] = rep.landmark_update
        out[prefix + f"pow_{tag}_order"] = rep.power_order_used
        out[prefix + f"pow_{tag}_trunc"] = rep.truncation_estimate
    return out


def make_mini():
    cfg_thr = solvers.SolverConfig(max_power_order=20, power_threshold=0.01)
    cfg_zero = solvers.SolverConfig(max_power_order=20, power_threshold=0.0)
    pose = objective.PoseConfig(0.1)
    for seed in range(3):
        problem = random_graph(5 + seed, 30 + 10 * seed, seed)
        rng = np.random.default_rng(100 + seed)
        cams = rng.standard_normal((problem.num_cameras, 3, 4))
        lms = np.concatenate([rng.standard_normal((problem.num_landmarks, 3)),
                              np.ones((problem.num_landmarks, 1))], axis=1)
        st1 = stratba.ProjectiveState(cams, lms)
        out = problem_arrays(problem)
        out["cams"], out["lms"] = cams, lms
        out["cost_s1"] = objective.total_cost(st1, problem, 1, pose)
        out["resolved"] = objective.solve_landmarks(st1, problem, pose)
        blocks = normal_eq.build_stage1_blocks(problem, st1, pose)
        probe12 = rng.standard_normal(problem.num_cameras * 12)
        for lam, mode, tag in ((1e-4, normal_eq.POSE_ONLY, "s1v_"), (0.3, normal_eq.BOTH, "s1j_")):
            system = normal_eq.assemble(blocks, lam, mode)
            out.update(system_arrays(tag, problem, system, cfg_thr, cfg_zero, probe12))
            out[tag + "lam"] = lam
        out["probe12"] = probe12
        # stage 2 on the retracted state
        st2 = riemannian.retract(st1)
        out["cams2"], out["lms2"] = st2.cameras, st2.landmarks
        out["cost_s2"] = objective.total_cost(st2, problem, 2)
        bases = riemannian.state_tangent_bases(st2)
        out["cam_bases"], out["lm_bases"] = bases.camera_bases, bases.landmark_bases
        raw = normal_eq.build_stage2_blocks(problem, st2)
        system2 = normal_eq.assemble(riemannian.project_blocks(raw, bases), 1e-3, normal_eq.BOTH)
        probe11 = rng.standard_normal(problem.num_cameras * 11)
        out["probe11"] = probe11
        out.update(system_arrays("s2_", problem, system2, cfg_thr, cfg_zero, probe11))
        out["s2_lam"] = 1e-3
        rep = riemannian.riemannian_step(problem, st2, cfg_thr, 1e-3, bases)
        trial = riemannian.apply_tangent_step(st2, bases, rep)
        out["s2_trial_cams"], out["s2_trial_lms"] = trial.cameras, trial.landmarks
        out["s2_trial_cost"] = objective.total_cost(trial, problem, 2)
        # short LM runs on the mini graph (both stages)
        for tag, stage, state, cfg in (
                ("lm1v_", 1, st1, solvers.SolverConfig(max_outer_iterations=15)),
                ("lm1j_", 1, st1, solvers.SolverConfig(max_outer_iterations=15, mode="joint")),
                ("lm2_", 2, st2, solvers.SolverConfig(max_outer_iterations=10))):
            final, trace = solvers.lm_minimize(problem, state, stage, cfg)
            out[tag + "costs"] = np.array([r.cost for r in trace.records])
            out[tag + "cams"], out[tag + "lms"] = final.cameras, final.landmarks
        np.savez_compressed(OUT / f"mini_{seed}.npz", **out)
        print("mini", seed, problem.num_observations)


def make_config_traces():
    pose = objective.PoseConfig(0.1)
    # tiny: stage 1 (20 its), then stage 2 from the lifted result
    problem, _ = synth.make_problem("tiny", 0)
    state = synth.random_state(problem, 1)
    st = stratba.ProjectiveState(state.cameras, state.landmarks)
    ref_problem = stratba.BaProblem(problem.num_cameras, problem.num_landmarks,
                                    problem.num_observations, problem.camera_indices,
                                    problem.landmark_indices, problem.measurements)
    out = problem_arrays(ref_problem)
    out["cams"], out["lms"] = st.cameras, st.landmarks
    cfg = solvers.SolverConfig(max_outer_iterations=20, max_power_order=20)
    blocks = normal_eq.build_stage1_blocks(ref_problem, st, pose)
    system = normal_eq.assemble(blocks, cfg.initial_lambda, normal_eq.POSE_ONLY)
    rep = solvers.power_schur_solve(system, cfg)
    out["it1_dx"], out["it1_dl"] = rep.pose_update, rep.landmark_update
    out["it1_order"], out["it1_trunc"] = rep.power_order_used, rep.truncation_estimate
    t = time.time()
    s1, tr1 = solvers.lm_minimize(ref_problem, st, 1, cfg)
    print("tiny stage1", time.time() - t)
    out["s1_costs"] = np.array([r.cost for r in tr1.records])
    out["s1_cams"], out["s1_lms"] = s1.cameras, s1.landmarks
    lifted = riemannian.lift_stage1_to_stage2(s1)
    out["s2_cams0"], out["s2_lms0"] = lifted.cameras, lifted.landmarks
    cfg2 = solvers.SolverConfig(max_outer_iterations=12)
    rep2 = riemannian.riemannian_step(ref_problem, lifted, cfg2, cfg2.initial_lambda)
    out["s2_it1_dx"], out["s2_it1_dl"] = rep2.pose_update, rep2.landmark_update
    out["s2_it1_order"] = rep2.power_order_used
    s2, tr2 = solvers.lm_minimize(ref_problem, lifted, 2, cfg2)
    out["s2_costs"] = np.array([r.cost for r in tr2.records])
    np.savez_compressed(OUT / "tiny_lm.npz", **out)

    problem, _ = synth.make_problem("small", 0)
    state = synth.random_state(problem, 1)
    ref_problem = stratba.BaProblem(problem.num_cameras, problem.num_landmarks,
                                    problem.num_observations, problem.camera_indices,
                                    problem.landmark_indices, problem.measurements)
    st = stratba.ProjectiveState(state.cameras, state.landmarks)
    t = time.time()
    _, tr = solvers.lm_minimize(ref_problem, st, 1, solvers.SolverConfig(max_outer_iterations=50))
    print("small stage1", time.time() - t)
    # the small problem itself is regenerated from the seeded generator; a
    # checksum pins it
    np.savez_compressed(OUT / "small_lm.npz", s1_costs=np.array([r.cost for r in tr.records]),
                        checksum=np.array([problem.num_observations,
                                           float(problem.measurements.sum()),
                                           float(problem.camera_indices.sum()),
                                           float(problem.landmark_indices.sum()),
                                           float(state.cameras.sum())]))


PCG_SETTINGS = (("t6", 1e-6, 500), ("t10", 1e-10, 5000), ("cap3", 1e-6, 3))


def pcg_arrays(prefix, system):
    out = {prefix + "diag": normal_eq.schur_diag_blocks(system)}
    for tag, tol, cap in PCG_SETTINGS:
        rep = solvers.pcg_schur_solve(system, solvers.SolverConfig(pcg_tolerance=tol,
                                                                   max_inner_iterations=cap))
        out[prefix + tag + "_dx"] = rep.pose_update
        out[prefix + tag + "_dl"] = rep.landmark_update
        out[prefix + tag + "_its"] = rep.inner_iterations_used
        out[prefix + tag + "_rel"] = rep.truncation_estimate
        out[prefix + tag + "_flag"] = rep.flag or ""
    return out


def make_pcg():
    pose = objective.PoseConfig(0.1)
    out = {}
    for seed in range(3):
        d = np.load(OUT / f"mini_{seed}.npz")
        problem = stratba.BaProblem(int(d["n_cameras"]), int(d["n_landmarks"]),
                                    len(d["cam_idx"]), d["cam_idx"].astype(np.int64),
                                    d["lm_idx"].astype(np.int64), d["meas"])
        st1 = stratba.ProjectiveState(d["cams"], d["lms"])
        blocks = normal_eq.build_stage1_blocks(problem, st1, pose)
        for lam, mode, tag in ((1e-4, normal_eq.POSE_ONLY, "s1v_"), (0.3, normal_eq.BOTH, "s1j_")):
            out.update(pcg_arrays(f"m{seed}_{tag}", normal_eq.assemble(blocks, lam, mode)))
        st2 = riemannian.retract(st1)
        bases = riemannian.state_tangent_bases(st2)
        raw = normal_eq.build_stage2_blocks(problem, st2)
        system2 = normal_eq.assemble(riemannian.project_blocks(raw, bases), 1e-3, normal_eq.BOTH)
        out.update(pcg_arrays(f"m{seed}_s2_", system2))
        for tag, stage, state in (("lm1_", 1, st1), ("lm2_", 2, st2)):
            cfg = solvers.SolverConfig(max_outer_iterations=10, inner_solver="pcg")
            final, trace = solvers.lm_minimize(problem, state, stage, cfg)
            out[f"m{seed}_{tag}costs"] = np.array([r.cost for r in trace.records])
            out[f"m{seed}_{tag}cams"] = final.cameras
            out[f"m{seed}_{tag}lms"] = final.landmarks
    # tiny config, stage 1 with the iterative solver (20 its)
    problem, _ = synth.make_problem("tiny", 0)
    state = synth.random_state(problem, 1)
    ref_problem = stratba.BaProblem(problem.num_cameras, problem.num_landmarks,
                                    problem.num_observations, problem.camera_indices,
                                    problem.landmark_indices, problem.measurements)
    st = stratba.ProjectiveState(state.cameras, state.landmarks)
    cfg = solvers.SolverConfig(max_outer_iterations=20, inner_solver="pcg")
    t = time.time()
    _, tr = solvers.lm_minimize(ref_problem, st, 1, cfg)
    print("tiny stage1 pcg", time.time() - t)
    out["tiny_lm1_costs"] = np.array([r.cost for r in tr.records])
    np.savez_compressed(OUT / "pcg.npz", **out)


if __name__ == "__main__":
    print("numpy", np.__version__)
    if sys.argv[1:] == ["pcg"]:
        make_pcg()
    else:
        make_mini()
        make_config_traces()
        make_pcg()

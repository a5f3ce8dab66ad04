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
    (20 its) and its first riemannian_step.
small_lm.npz -- BASELINE small config: reference stage-1 cost trace (50 its).
pcg.npz      -- the PCG inner solver (solvers.py:153-187) on the mini graphs:
    schur_diag_blocks and pcg_schur_solve at three (tolerance, cap) settings for
    the stage-1 varpro / joint and stage-2 systems, plus lm_minimize traces with
    inner_solver="pcg" (stage 1 and 2) on the mini graphs and the tiny config.

bal_cases.json -- parse_bal outcomes (arrays or BalParseError line + message) on
    hand-written texts covering the token grammar and every error path.
tiny.bal.gz  -- the tiny config written by the reference's write_bal (parser and
    pipeline input); prune.npz -- prune_underobserved on a graph with single,
    duplicate-camera and unobserved landmarks and an empty camera.
pipeline_*   -- run_problem summaries / trace CSVs on tiny.bal.gz
    (povar + ripoba full, iterative stage 1).

spectral.npz -- spectral_check (solvers.py:263-295) on the mini systems, with the dense top
    eigenvalue of U^-1 W V^+ W^T beside it.

``python tests/golden/make_golden.py pcg|bal|spectral|traces`` regenerates one group only.
Scale and edge-case fixtures: tests/golden/make_golden_scale.py.
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
    cfg2 = solvers.SolverConfig(max_outer_iterations=20)
    rep2 = riemannian.riemannian_step(ref_problem, lifted, cfg2, cfg2.initial_lambda)
    out["s2_it1_dx"], out["s2_it1_dl"] = rep2.pose_update, rep2.landmark_update
    out["s2_it1_order"] = rep2.power_order_used
    s2, tr2 = solvers.lm_minimize(ref_problem, lifted, 2, cfg2)
    out["s2_costs"] = np.array([r.cost for r in tr2.records])
    # the default tolerance stops stage 2 after a few iterations; all 20 (north_star)
    cfg20 = solvers.SolverConfig(max_outer_iterations=20, function_tolerance=1e-300)
    _, tr20 = solvers.lm_minimize(ref_problem, lifted, 2, cfg20)
    out["s2_costs20"] = np.array([r.cost for r in tr20.records])
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


def make_spectral():
    """spectral.npz: the reference's spectral_check (solvers.py:263-295) and the dense top
    eigenvalue of U^-1 W V^+ W^T on the mini systems (stage-1 varpro / joint, stage 2)."""
    pose = objective.PoseConfig(0.1)
    out = {}
    for seed in range(3):
        d = np.load(OUT / f"mini_{seed}.npz")
        problem = stratba.BaProblem(int(d["n_cameras"]), int(d["n_landmarks"]),
                                    len(d["cam_idx"]), d["cam_idx"].astype(np.int64),
                                    d["lm_idx"].astype(np.int64), d["meas"])
        st1 = stratba.ProjectiveState(d["cams"], d["lms"])
        blocks = normal_eq.build_stage1_blocks(problem, st1, pose)
        systems = [(tag, normal_eq.assemble(blocks, lam, mode))
                   for lam, mode, tag in ((1e-4, normal_eq.POSE_ONLY, "s1v_"),
                                          (0.3, normal_eq.BOTH, "s1j_"))]
        st2 = riemannian.retract(st1)
        bases = riemannian.state_tangent_bases(st2)
        raw = normal_eq.build_stage2_blocks(problem, st2)
        systems.append(("s2_", normal_eq.assemble(riemannian.project_blocks(raw, bases), 1e-3,
                                                  normal_eq.BOTH)))
        for tag, system in systems:
            out[f"m{seed}_{tag}mu"] = solvers.spectral_check(system)
            out[f"m{seed}_{tag}mu3000"] = solvers.spectral_check(system, max_iterations=3000)
            u = np.zeros((system.pose_dim, system.pose_dim))
            d_ = system.u_blocks.shape[1]
            for i in range(system.n_cameras):
                u[i * d_:(i + 1) * d_, i * d_:(i + 1) * d_] = system.u_blocks[i]
            cols = np.stack([solvers._coupling_round_trip(system, e)
                             for e in np.eye(system.pose_dim)], axis=1)
            m = np.linalg.solve(u, cols)
            out[f"m{seed}_{tag}dense"] = float(np.max(np.real(np.linalg.eigvals(m))))
    np.savez_compressed(OUT / "spectral.npz", **out)
    print("spectral", {k: v for k, v in out.items() if k.endswith("mu")})


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


BAL_TEXTS = {
    "basic": "2 3 4\n0 0 1.5 -2\n1 0 3e-1 4E+2\n0 1 5 6\n1 2 7 8\n"
             + "1 2 3 4 5 6 7 8 9\n" * 2 + "0.1 0.2 0.3\n" * 3,
    "whitespace": "2\t3  4\r\n0 0\r1.5 -2 1 0\v3e-1\f4E+2\n\n0 1 5 6 1 2 7\u00a08\n"
                  + " ".join(["1"] * 18) + "\r\n" + " ".join(["0.5"] * 9) + "\n",
    "syntax": "+2 0_3 004\n00 0_1 1_000.5 .5\n1 0 5. -.25e-1_0\n0 1 1e-400 1e400\n"
              "1 2 inf -Infinity\n" + "1 2 3 4 5 6 7 8 9\n" * 2 + "0.1 0.2 0.3\n" * 3,
    "empty": "",
    "header_float": "2.0 3 4\n",
    "header_negative": "2 -3 4\n",
    "header_truncated": "2 3",
    "cam_range": "2 3 1\n2 0 1 1\n",
    "pt_range": "2 3 1\n\n1 -1 1 1\n",
    "big_index": "2 3 1\n99999999999999999999 0 1 1\n",
    "int_as_float": "2 3 1\n1e0 0 1 1\n",
    "bad_underscore": "2 3 1\n1__0 0 1 1\n",
    "bad_meas": "2 3 1\n1 0 abc 1\n",
    "quote_token": "2 3 1\n1 0 1 a'b\n",
    "obs_truncated": "2 3 2\n1 0 1 1\n0 1\n",
    "cam_truncated": "1 1 1\n0 0 1 1\n1 2 3\n",
    "pt_truncated": "1 1 1\n0 0 1 1\n1 2 3 4 5 6 7 8 9\n1 2\n",
    "trailing": "1 1 1\n0 0 1 1\n1 2 3 4 5 6 7 8 9\n1 2 3\n\n4\n",
    "bad_cam_param": "1 1 1\n0 0 1 1\n1 2 3 4 x 6 7 8 9\n1 2 3\n",
    "hex_float": "1 1 1\n0 0 0x1p3 1\n",
}


def make_bal():
    import gzip
    import io
    import json
    from stratba import bal_io
    cases = []
    for name, text in BAL_TEXTS.items():
        try:
            p = bal_io.parse_bal(io.StringIO(text))
            out = {"ok": {"n": [p.num_cameras, p.num_landmarks, p.num_observations],
                          "cam": p.camera_indices.tolist(), "pt": p.landmark_indices.tolist(),
                          "meas": [[repr(float(v)) for v in r] for r in p.measurements],
                          "cams": [[repr(float(v)) for v in r] for r in p.metric_cameras],
                          "pts": [[repr(float(v)) for v in r] for r in p.metric_points]}}
        except bal_io.BalParseError as exc:
            out = {"error": [exc.line, str(exc)]}
        cases.append({"name": name, "text": text, **out})
    with open(OUT / "bal_cases.json", "w") as fh:
        json.dump(cases, fh, indent=1)
    # tiny config through the reference writer
    problem, _ = synth.make_problem("tiny", 0)
    ref_problem = stratba.BaProblem(problem.num_cameras, problem.num_landmarks,
                                    problem.num_observations, problem.camera_indices,
                                    problem.landmark_indices, problem.measurements)
    buf = io.StringIO()
    bal_io.write_bal(ref_problem, buf)
    with gzip.GzipFile(OUT / "tiny.bal.gz", "wb", mtime=0) as fh:
        fh.write(buf.getvalue().encode())
    # pruning: singles, a duplicate-camera landmark, an unobserved landmark, an empty camera
    rng = np.random.default_rng(7)
    ci, li = [], []
    for j in range(40):
        kind = j % 5
        if kind == 0:      # single observation
            cams = [int(rng.integers(0, 6))]
        elif kind == 1:    # same camera twice
            c = int(rng.integers(0, 6))
            cams = [c, c]
        elif kind == 2:    # unobserved
            cams = []
        else:
            cams = sorted(rng.choice(6, size=int(rng.integers(2, 5)), replace=False).tolist())
        for c in cams:
            ci.append(c)
            li.append(j)
    ci = np.array(ci)
    ci[ci == 4] = 5  # camera 4 only ever sees pruned landmarks / nothing
    perm = rng.permutation(len(ci))
    meas = rng.standard_normal((len(ci), 2))
    raw = stratba.BaProblem(7, 40, len(ci), ci[perm], np.array(li)[perm], meas,
                            rng.standard_normal((7, 9)), rng.standard_normal((40, 3)))
    pr = bal_io.prune_underobserved(raw)
    np.savez_compressed(OUT / "prune.npz", cam_idx=raw.camera_indices, lm_idx=raw.landmark_indices,
                        meas=raw.measurements, cams=raw.metric_cameras, pts=raw.metric_points,
                        p_n=np.array([pr.num_cameras, pr.num_landmarks, pr.num_observations]),
                        p_cam=pr.camera_indices, p_lm=pr.landmark_indices, p_meas=pr.measurements,
                        p_cams=pr.metric_cameras, p_pts=pr.metric_points)
    # the pipeline on tiny.bal.gz
    import shutil
    import tempfile
    from stratba import pipeline
    # seed 0 / 30 iterations: a stage-1 result converged enough for a well-conditioned
    # stage 2 (the oracle reproduces this chain within 3e-11); the PCG chain is
    # tolerance-limited, so its fixture covers stage 1 only
    for tag, stage, s1, s2, its in (("povar", "full", "povar", "ripoba", 30),
                                    ("iterative", "stage1", "iterative", "ripcg", 20)):
        with tempfile.TemporaryDirectory() as td:
            spec = pipeline.RunSpec(inputs=[str(OUT / "tiny.bal.gz")], seed=0, stage=stage,
                                    stage1_solver=s1, stage2_solver=s2, max_iterations=its,
                                    out_dir=td)
            pipeline.run_problem(OUT / "tiny.bal.gz", spec)
            shutil.copy(Path(td) / "tiny_summary.json", OUT / f"pipeline_{tag}_summary.json")
            shutil.copy(Path(td) / "tiny_trace.csv", OUT / f"pipeline_{tag}_trace.csv")
        print("pipeline", tag)


if __name__ == "__main__":
    print("numpy", np.__version__)
    if sys.argv[1:] == ["pcg"]:
        make_pcg()
    elif sys.argv[1:] == ["spectral"]:
        make_spectral()
    elif sys.argv[1:] == ["bal"]:
        make_bal()
    elif sys.argv[1:] == ["traces"]:
        make_config_traces()
    else:
        make_mini()
        make_config_traces()
        make_pcg()
        make_bal()

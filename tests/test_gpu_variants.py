"""Kernel variants selected by pv_set_option knobs give the same results (needs a B200).

The persistent TMA-pipelined camera kernel (PV_OPT_CAM_PIPE, pv_pipe.cuh) runs when the
landmark blocks are small enough for one warp per camera (wpc == 1, the vlarge case);
there it must reproduce k_cam bit for bit, and both must match the reference's golden
step and 20-iteration cost trace (tests/golden/tiny_lm.npz) within the north_star's
tolerances.
"""

import numpy as np
import pytest

from _pvutil import golden, problem_from, rel

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pv():
    import paper_2405_05079_b200 as pv
    return pv


def _ctx(pv, z, knobs):
    from paper_2405_05079_b200 import _lib
    dp = pv.DeviceProblem(problem_from(z), 0.1)
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)  # 4 landmark blocks: one warp per camera
    for k, v in knobs:
        dp.set_option(k, v)
    return dp


@pytest.mark.parametrize("stage", [1, 2])
def test_pipe_matches_k_cam(pv, stage):
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    st = pv.ProjectiveState(z["cams"], z["lms"]) if stage == 1 else \
        pv.ProjectiveState(z["s2_cams0"], z["s2_lms0"])
    outs = []
    # the term graph (default), the host term loop, the one-kernel series (k_series), the
    # full (x, m) stream, and the contiguous work-list balance, all against k_cam
    variants = ([(_lib.PV_OPT_CAM_PIPE, 0)], [(_lib.PV_OPT_CAM_PIPE, 1)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_XM, 0)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_GRAPH, 0)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_SERIES, 1)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_SERIES, 1), (_lib.PV_OPT_XM, 0)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_BALANCE, 0)],
                [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_SERIES, 1), (_lib.PV_OPT_BALANCE, 0)])
    for knobs in variants:
        dp = _ctx(pv, z, knobs)
        info = dp.info()
        assert info["blocks"] > 1 and info["warps_per_cam"] == 1
        if stage == 1:
            sysm = pv.assemble_system(dp.problem, st, 1, 1e-4, "pose_only", dp=dp)
            rep = pv.power_schur_solve(sysm, pv.SolverConfig())
        else:
            rep = pv.riemannian_step(dp.problem, st, pv.SolverConfig(), dp=dp)
        outs.append(rep)
    a = outs[0]
    for b in outs[1:]:
        assert b.power_order_used == a.power_order_used
        np.testing.assert_array_equal(b.pose_update, a.pose_update)
        np.testing.assert_array_equal(b.landmark_update, a.landmark_update)
    key = "it1_" if stage == 1 else "s2_it1_"
    assert a.power_order_used == int(z[key + "order"])
    # stage 2: the reduced RHS is a cancellation (tests/test_gpu_parity.py uses 1e-8 too)
    tol = 1e-10 if stage == 1 else 1e-8
    assert rel(a.pose_update, z[key + "dx"]) <= tol
    if stage == 1:
        assert rel(a.landmark_update, z[key + "dl"]) <= tol


def test_compact_stream_falls_back_when_w_is_not_one(pv):
    """The compact stage-1 stream (PV_OPT_XM) drops the landmark's w = 1; a stage-1 state
    whose landmarks do not all have w = 1 (the reference uses the full 4-vector,
    objective.py:68-110) must take the full stream and still match k_cam bit for bit."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    lms = np.array(z["lms"])
    lms[::7, 3] = 1.5
    st = pv.ProjectiveState(z["cams"], lms)
    outs = []
    for knobs in ([(_lib.PV_OPT_CAM_PIPE, 0)], [(_lib.PV_OPT_CAM_PIPE, 1)]):
        dp = _ctx(pv, z, knobs)
        sysm = pv.assemble_system(dp.problem, st, 1, 1e-4, "pose_only", dp=dp)
        outs.append(pv.power_schur_solve(sysm, pv.SolverConfig()))
    assert outs[0].power_order_used == outs[1].power_order_used
    np.testing.assert_array_equal(outs[0].pose_update, outs[1].pose_update)
    np.testing.assert_array_equal(outs[0].landmark_update, outs[1].landmark_update)


@pytest.mark.parametrize("series", [0, 1])
def test_pipe_lm_trace_matches_reference(pv, series):
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    dp = _ctx(pv, z, [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_SERIES, series)])
    st = pv.ProjectiveState(z["cams"], z["lms"])
    _, trace = pv.lm_minimize(dp.problem, st, 1, pv.SolverConfig(max_outer_iterations=20),
                              dp=dp)
    c = np.array([r.cost for r in trace.records])
    ref = z["s1_costs"]
    assert len(c) == len(ref)
    np.testing.assert_allclose(c, ref, rtol=1e-6, atol=0)
    assert "".join("a" if y < x else "r" for x, y in zip(c, c[1:])) == \
        "".join("a" if y < x else "r" for x, y in zip(ref, ref[1:]))


@pytest.mark.parametrize("stage", [1, 2])
def test_pipe_long_work_lists_large(pv, stage):
    """The large config with 8 MB landmark blocks: one warp per camera, ~75 work items per
    warp (the descriptor window of k_cam_pipe shifts several times); the pipelined camera
    pass must reproduce k_cam bit for bit through a power solve and back-substitution."""
    from paper_2405_05079_b200 import _lib, synth
    problem, _ = synth.make_problem("large", 0)
    dp = pv.DeviceProblem(problem, 0.1)
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 8 << 20)
    st = synth.random_state(problem, 1)
    if stage == 2:  # a stage-1 state first, then the lifted projective state
        st, _ = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=2), dp=dp)
        st = pv.lift_stage1_to_stage2(st)
    dp.set_state(st)
    dp.linearize(stage)
    dp.damp(1e-4, stage == 2)
    assert dp.info()["warps_per_cam"] == 1 and dp.info()["blocks"] > 10
    out = []
    for v, series in ((0, 0), (1, 0), (1, 1)):  # k_cam, launch per block, series kernel
        dp.set_option(_lib.PV_OPT_CAM_PIPE, v)
        dp.set_option(_lib.PV_OPT_SERIES, series)
        dp.linearize(stage)
        dp.damp(1e-4, stage == 2)
        order, trunc = dp.power_solve(4, 0.0)
        dx, dl = dp.step(stage)
        out.append((order, trunc, dx.copy(), dl.copy()))
    for o in out[1:]:
        assert out[0][0] == o[0] == 4 and out[0][1] == o[1]
        np.testing.assert_array_equal(out[0][2], o[2])
        np.testing.assert_array_equal(out[0][3], o[3])


@pytest.mark.parametrize("slots", [0, 1])
def test_resolve_and_landmark_linearization_variants(pv, slots):
    """PV_OPT_RESOLVE_SLOTS: lane-per-landmark slots (1, default) or warp-per-task (0) for the
    landmark re-solve and the landmark side of the linearization; both reproduce the
    reference's 20-iteration stage-1 trace and its first stage-2 step (tiny config)."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    dp = pv.DeviceProblem(problem_from(z), 0.1)
    dp.set_option(_lib.PV_OPT_RESOLVE_SLOTS, slots)
    st = pv.ProjectiveState(z["cams"], z["lms"])
    _, trace = pv.lm_minimize(dp.problem, st, 1, pv.SolverConfig(max_outer_iterations=20),
                              dp=dp)
    c = np.array([r.cost for r in trace.records])
    np.testing.assert_allclose(c, z["s1_costs"], rtol=1e-6, atol=0)
    rep = pv.riemannian_step(dp.problem, pv.ProjectiveState(z["s2_cams0"], z["s2_lms0"]),
                             pv.SolverConfig(), dp=dp)
    assert rep.power_order_used == int(z["s2_it1_order"])
    assert rel(rep.pose_update, z["s2_it1_dx"]) <= 1e-8


@pytest.mark.parametrize("solver", ["power", "pcg"])
def test_rhs_reuse_after_rejected_step(pv, solver):
    """PV_OPT_RHS_REUSE: a second solve on the same POSE_ONLY linearization (a rejected step
    retried with larger damping) reuses the reduced RHS; the steps are bit-identical to
    recomputing it, and a BOTH-damped solve in between invalidates the reuse."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    out = []
    for reuse in (0, 1):
        dp = pv.DeviceProblem(problem_from(z), 0.1)
        dp.set_option(_lib.PV_OPT_RHS_REUSE, reuse)
        dp.set_state(pv.ProjectiveState(z["cams"], z["lms"]))
        dp.linearize(1)
        steps = []
        for lam, both in ((1e-4, False), (4e-4, False), (1.6e-3, True), (6.4e-3, False)):
            dp.damp(lam, both)
            if solver == "power":
                dp.power_solve(20, 0.01)
            else:
                dp.pcg_solve(50, 1e-8)
            steps.append(np.concatenate(dp.step(1)))
        out.append(steps)
    for a, b in zip(*out):
        np.testing.assert_array_equal(a, b)


def test_reblocking_keeps_damped_landmark_inverse(pv):
    """V+ and t live in warp-slot order (build_ktasks); a re-blocking after pv_damp
    (PV_OPT_BLOCK_BYTES) moves V+ to the new slot positions: the debug view is unchanged, and
    after the re-linearization the re-blocking requires, the solve equals the one on a
    context blocked that way from the start."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    st = pv.ProjectiveState(z["cams"], z["lms"])
    outs = []
    for late in (False, True):
        dp = pv.DeviceProblem(problem_from(z), 0.1)
        if not late:
            dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
        dp.set_state(st)
        dp.linearize(1)
        dp.damp(1e-4, True)
        vp0 = dp.debug(_lib.PV_DBG_VPINV).copy()
        if late:
            dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
            np.testing.assert_array_equal(dp.debug(_lib.PV_DBG_VPINV), vp0)
        assert dp.info()["blocks"] > 1
        dp.linearize(1)  # a re-blocking drops the camera-sorted copies of the state
        dp.damp(1e-4, True)
        np.testing.assert_array_equal(dp.debug(_lib.PV_DBG_VPINV), vp0)
        dp.power_solve(20, 0.01)
        outs.append(np.concatenate(dp.step(1)))
    np.testing.assert_array_equal(outs[0], outs[1])


@pytest.mark.parametrize("block_bytes", [64 << 10, 80 << 20])
def test_cost_camera_sorted_matches_task_order(pv, block_bytes):
    """pv_cost over the camera-sorted segments (PV_OPT_COST_CS, k_cost_cs) and over the
    landmark tasks (k_cost) sum the same per-observation terms in different fixed orders:
    equal to rounding, and both equal the oracle's total_cost (objective.py:194-211) on the
    golden starts of tests/golden/tiny_lm.npz."""
    from oracle import povar_oracle as O
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    starts = {1: (z["cams"], z["lms"]), 2: (z["s2_cams0"], z["s2_lms0"])}
    g = O.graph_of(problem_from(z))
    for stage, (cams, lms) in starts.items():
        want = O.total_cost(g, cams, lms, stage)
        got = []
        for knob in (0, 1):
            dp = pv.DeviceProblem(problem_from(z), 0.1)
            dp.set_option(_lib.PV_OPT_BLOCK_BYTES, block_bytes)
            dp.set_option(_lib.PV_OPT_COST_CS, knob)
            dp.set_state(pv.ProjectiveState(cams, lms))
            got.append(dp.cost(stage))
        assert got[1] == pytest.approx(got[0], rel=1e-13, abs=0)
        assert got[1] == pytest.approx(want, rel=1e-12, abs=0)


def test_cost_camera_sorted_degenerate_depth(pv):
    """A stage-2 observation with |z| <= 1e-12 makes the camera-sorted cost +inf, as
    total_cost does (objective.py:206-210)."""
    from paper_2405_05079_b200 import _lib
    import _kat
    pr, st, _ = _kat.degenerate_depth_case()
    dp = pv.DeviceProblem(pr, 0.1)
    dp.set_option(_lib.PV_OPT_COST_CS, 1)
    dp.set_state(st)
    assert dp.cost(2) == np.inf


@pytest.mark.parametrize("max_order,thr", [(20, 0.01), (20, 0.0), (3, 0.0), (1, 0.01)])
def test_graph_term_loop_matches_host_loop(pv, max_order, thr):
    """PV_OPT_GRAPH: the term loop as a CUDA graph WHILE node (device-side stop test) gives
    the host loop's order, truncation and steps bit for bit -- stop by threshold, by the order
    cap, and a one-term series; and the captured graph is reused across solves."""
    from paper_2405_05079_b200 import _lib
    z = golden("tiny_lm.npz")
    st = pv.ProjectiveState(z["cams"], z["lms"])
    outs = []
    for graph in (0, 1):
        dp = _ctx(pv, z, [(_lib.PV_OPT_GRAPH, graph)])
        sysm = pv.assemble_system(dp.problem, st, 1, 1e-4, "pose_only", dp=dp)
        cfg = pv.SolverConfig(max_power_order=max_order, power_threshold=thr)
        reps = [pv.power_schur_solve(sysm, cfg) for _ in range(2)]
        assert reps[0].power_order_used == reps[1].power_order_used
        np.testing.assert_array_equal(reps[0].pose_update, reps[1].pose_update)
        outs.append(reps[0])
    a, b = outs
    assert a.power_order_used == b.power_order_used
    assert a.truncation_estimate == b.truncation_estimate
    np.testing.assert_array_equal(a.pose_update, b.pose_update)
    np.testing.assert_array_equal(a.landmark_update, b.landmark_update)
    if thr == 0.0:
        assert a.power_order_used == max_order


@pytest.mark.parametrize("block_kb", [1 << 20, 176, 120])
def test_few_blocks_many_cameras_all_term_paths(pv, block_kb):
    """600 cameras x 2,500 landmarks (about 16 observations per camera): one warp per camera
    even with a single landmark block, so the pipelined kernel, the term graph and the
    one-kernel series all run with B = 1, 2 and 3 blocks (the series' first and last steps
    drop their out-of-range parts) -- each must reproduce k_cam bit for bit, stage 1 and 2,
    with tracks longer than a warp slot present (power-law lengths up to 150)."""
    from paper_2405_05079_b200 import _lib, synth
    cfg = synth.SynthConfig("wide", 600, 2500, ("power", 4.0, 150))
    problem, _ = synth.make_problem(cfg, 3)
    st1 = synth.random_state(problem, 2)
    for stage in (1, 2):
        st = st1 if stage == 1 else pv.lift_stage1_to_stage2(st1)
        outs, blocks = [], None
        for knobs in ([(_lib.PV_OPT_CAM_PIPE, 0)], [(_lib.PV_OPT_CAM_PIPE, 1)],
                      [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_GRAPH, 0)],
                      [(_lib.PV_OPT_CAM_PIPE, 1), (_lib.PV_OPT_SERIES, 1)]):
            dp = pv.DeviceProblem(problem, 0.1)
            dp.set_option(_lib.PV_OPT_BLOCK_BYTES, block_kb << 10)
            for k, v in knobs:
                dp.set_option(k, v)
            info = dp.info()
            assert info["warps_per_cam"] == 1
            blocks = info["blocks"]
            dp.set_state(st)
            dp.linearize(stage)
            dp.damp(1e-4, stage == 2)
            order, trunc = dp.power_solve(6, 0.0)
            dx, dl = dp.step(stage)
            outs.append((order, trunc, dx.copy(), dl.copy()))
        assert blocks == {1 << 20: 1, 176: 2, 120: 3}[block_kb], blocks
        for o in outs[1:]:
            assert o[0] == outs[0][0] == 6 and o[1] == outs[0][1]
            np.testing.assert_array_equal(o[2], outs[0][2])
            np.testing.assert_array_equal(o[3], outs[0][3])


@pytest.mark.parametrize("config", ["small", "large"])
def test_slot_records_match_lane_entries(pv, config):
    """PV_OPT_KSLOT: the stage-1 term reduce reading one 16-byte record per warp slot gives
    the per-lane entries' series bit for bit, in the host loop and in the term graph (small:
    20 track lengths per block, partly filled slots; large: tracks longer than a 64-observation
    slot, reduced by a whole warp)."""
    from paper_2405_05079_b200 import _lib, synth
    problem, _ = synth.make_problem(config, 0)
    dp = pv.DeviceProblem(problem, 0.1)
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, (64 << 10) if config == "small" else (8 << 20))
    dp.set_state(synth.random_state(problem, 1))
    out = []
    for kslot, graph in ((0, 0), (1, 0), (1, 1)):
        dp.set_option(_lib.PV_OPT_KSLOT, kslot)
        dp.set_option(_lib.PV_OPT_GRAPH, graph)
        dp.linearize(1)
        dp.damp(1e-4, False)
        order, trunc = dp.power_solve(6, 0.0)
        dx, dl = dp.step(1)
        out.append((order, trunc, dx.copy(), dl.copy()))
    for o in out[1:]:
        assert out[0][0] == o[0] == 6 and out[0][1] == o[1]
        np.testing.assert_array_equal(out[0][2], o[2])
        np.testing.assert_array_equal(out[0][3], o[3])

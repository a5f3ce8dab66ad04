"""PoVar hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[4], the config the metric's target is quoted
on; it fits one B200): the seeded 13,682-camera / 4,456,117-landmark /
~29.0M-observation synthetic problem, fp64, stage-1 PoVar (varpro + power
series, <= 30 terms, threshold 0.01), random N(0,1) start.

* a "step" = one full stage-1 LM iteration (linearize, damp, power series,
  back-substitution, trial, cost, accept + closed-form landmark re-solve)
  continuing an LM run; ``value`` = n_obs x iterations/s (obs/s), inputs
  resident in HBM.
* ``spmv`` = the S'.v term alone (the power-series unit of work).
* ``roofline`` = the dominant term kernel, algorithmic bytes / mean launch
  time from CUDA events inside this run.
* ``e2e`` = the public ``lm_minimize`` call with host state in / out
  (one iteration per call), i.e. host<->device copies inside the timing.
* ``--impl reference`` times the CPU oracle port (oracle/povar_oracle.py, the
  NumPy restatement of the reference) on a landmark-subsampled slice.

Multi-GPU: ``torchrun --nproc-per-node N bench.py --gpus N``: landmarks are
sharded across ranks (equal observation counts), cameras replicated, one NCCL
allreduce of the camera vector per term; timings are max over ranks.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "power-series S'x mat-vecs/s and LM iters/s (obs/s); % of HBM roofline"
CONFIG = "vlarge"
CPU_SAMPLE_FRACTION = 0.01  # landmark fraction of vlarge timed on the CPU (~290k obs)


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def term_bytes(n_p, n_l, n_o, stage=1):
    """Algorithmic bytes of one power-series term per kernel.

    Every array element a kernel must touch, counted once per pass.  k_cam
    (summed over the landmark blocks) streams the camera-sorted x (32), m (16)
    and one id (4) twice -- once for W t, once for W^T v -- scatters s (32) and
    reads each landmark's t once (32 per landmark), plus per camera P, U^-1 and
    the small vectors (~1.6 KB).  k_lm_reduce reads s (32 per observation) and
    per landmark its work-slot entry (16), V+ (2 x 32 B sectors), x (stage 2) and
    writes t (32).  s and t are sized per block to stay in the persisting L2,
    so the DRAM-compulsory part is the streams + per-landmark data.
    """
    lmr = 32 * n_o + (112 if stage == 1 else 144) * n_l
    cam = 136 * n_o + 32 * n_l + 1600 * n_p
    r1 = (292 if stage == 1 else 268) * n_o + 52 * n_l + (1632 if stage == 1 else 1408) * n_p
    return {"lm_reduce": lmr, "cam": cam, "r1_term": r1}


def traffic_from_profile(kernel, n_o):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture (vlarge only)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f)
        if t.get("n_obs") == n_o:
            return t["per_term_bytes"].get(kernel)
    except Exception:
        pass
    return None


def cpu_port_lm(fraction, iters=2, seed=0):
    """Time the oracle port (NumPy restatement of the reference) on a slice."""
    from oracle import povar_oracle as O
    from paper_2405_05079_b200 import synth
    problem, _ = synth.make_problem(CONFIG, seed, landmark_fraction=fraction)
    state = synth.random_state(problem, 1)
    g = O.graph_of(problem)
    cams, lms = np.array(state.cameras), np.array(state.landmarks)
    O.lm_minimize(g, cams, lms, 1, max_iterations=1, max_order=30, ftol=1e-300)  # warm
    t = time.perf_counter()
    log = O.lm_minimize(g, cams, lms, 1, max_iterations=iters, max_order=30, ftol=1e-300)
    dt = (time.perf_counter() - t) / max(1, len(log.decisions))
    return problem.num_observations / dt, dt, problem


def run_reference(args, rank, world):
    if rank != 0:
        return
    fr = CPU_SAMPLE_FRACTION
    from oracle import povar_oracle as O
    from paper_2405_05079_b200 import synth
    problem, _ = synth.make_problem(CONFIG, 0, landmark_fraction=fr)
    state = synth.random_state(problem, 1)
    g = O.graph_of(problem)
    cams, lms = np.array(state.cameras), np.array(state.landmarks)
    # warmup + timed LM iterations of the NumPy port, continuing one LM run
    log = O.lm_minimize(g, cams, lms, 1, max_iterations=max(1, args.warmup), max_order=30,
                        ftol=1e-300)
    cams, lms = log.cams, log.lms
    t = time.perf_counter()
    log = O.lm_minimize(g, cams, lms, 1, max_iterations=args.steps, max_order=30, ftol=1e-300)
    dt = time.perf_counter() - t
    n_it = len(log.decisions)
    value = problem.num_observations * n_it / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "obs/s",
            "n_gpus": world, "steps": n_it, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / n_it, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE vlarge generator, landmark-subsampled)",
            "config": {"workload": "vlarge stage-1 PoVar LM iteration (CPU oracle port)",
                       "landmark_fraction": fr, "n_cameras": problem.num_cameras,
                       "n_landmarks": problem.num_landmarks,
                       "n_obs": problem.num_observations, "max_power_order": 30},
            "cpu_baseline": {"value": value, "unit": "obs/s", "cores": 1, "kind": "port",
                             "sample": f"{fr:.0%} of vlarge landmarks "
                                       f"({problem.num_observations} obs), {n_it} LM iterations"},
            "e2e": {"value": value, "unit": "obs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default=CONFIG)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-stage2", action="store_true")
    ap.add_argument("--no-pcg", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist

    import paper_2405_05079_b200 as pv
    from paper_2405_05079_b200 import shard, synth

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    cfg = synth.CONFIGS[args.config]
    problem, _ = synth.make_problem(args.config, 0)
    state0 = synth.random_state(problem, 1)
    n_p, n_l, n_o = problem.num_cameras, problem.num_landmarks, problem.num_observations
    plan = shard.plan_shards(problem, world)
    nccl_id = shard.broadcast_nccl_id(rank, world) if world > 1 else None
    dp = pv.DeviceProblem(problem, 0.1, device=local, rank=rank, world=world, nccl_id=nccl_id,
                          lm_range=plan[rank])
    stream = torch.cuda.ExternalStream(dp.stream_handle, device=local)
    scfg = pv.SolverConfig(max_outer_iterations=1, max_power_order=cfg.max_power_order,
                           function_tolerance=1e-300)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- LM iterations (value) -------------------------------------------------
    dp.set_state(state0)
    f = dp.cost(1)
    lam = scfg.initial_lambda
    orders = []

    linearized = [False]

    def lm_iteration():
        # solver.lm_minimize's iteration: a rejected step leaves the state unchanged, so its
        # linearization (and, POSE_ONLY, the reduced RHS) is reused
        nonlocal f, lam
        if not linearized[0]:
            dp.linearize(1)
            linearized[0] = True
        dp.damp(lam, False)
        order, _ = dp.power_solve(scfg.max_power_order, scfg.power_threshold)
        orders.append(order)
        ok = dp.trial(1)
        ft = dp.cost(1, trial=True) if ok else math.inf
        if ft < f:
            f, _ = dp.accept(1, resolve=True)
            linearized[0] = False
            lam = max(scfg.lambda_min, lam * scfg.lambda_decrease)
        else:
            lam = min(scfg.lambda_max, lam * scfg.lambda_increase)

    for _ in range(args.warmup):
        lm_iteration()
    orders.clear()
    launches0 = dp.info()["launches"]
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            lm_iteration()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    launches = dp.info()["launches"] - launches0
    ms_step = ms_total / args.steps
    value = n_o * args.steps / (ms_total * 1e-3)

    # ---- S'.v terms and per-kernel roofline ------------------------------------
    dp.linearize(1)
    dp.damp(lam, False)
    dp.power_solve(1, 0.0)
    dp.bench_terms(1, 3)
    barrier()
    kt = dp.bench_terms(1, 20)
    kt = {k: max_over_ranks(v) for k, v in kt.items()}
    peak, peak_src = _peaks()
    loc = dp.info()
    tb = term_bytes(n_p, loc["n_l_local"], loc["n_o_local"], 1)
    kern = {}
    # one warp per camera: the persistent TMA-pipelined camera kernel runs the blocks
    cam_name = "k_cam_pipe" if loc["warps_per_cam"] == 1 else "k_cam"
    for name, key, tkey in (("k_lm_reduce", "lm_reduce", "phase1_ms"),
                            (cam_name, "cam", "phase2_ms")):
        ms = kt[tkey]
        gbs = tb[key] / (ms * 1e-3) / 1e9
        kern[name] = {"ms": ms, "algorithmic_bytes": tb[key], "achieved_gbs": gbs,
                      "frac": gbs / peak}
    dom = max(kern, key=lambda k: kern[k]["ms"])
    term_ms = kt["term_ms"]
    spmv = {"ms_per_term": term_ms, "terms_per_s": 1e3 / term_ms,
            "obs_per_s": n_o / (term_ms * 1e-3),
            "r1_equivalent_gbs": tb["r1_term"] * world / (term_ms * 1e-3) / 1e9,
            "r1_equivalent_frac": tb["r1_term"] * world / (term_ms * 1e-3) / 1e9 / peak,
            "r1_equivalent_frac_of_8tbs": tb["r1_term"] * world / (term_ms * 1e-3) / 8e12,
            "kernels": kern}
    roofline = {"bound": "hbm", "achieved": kern[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["frac"],
                "traffic": traffic_from_profile(dom, n_o), "kernel": dom,
                "peak_source": peak_src,
                "note": "achieved/traffic per term (summed over the landmark-block launches)"}

    # ---- PCG inner solver ("iterative", solvers.py:153-187) on the same system -----
    pcg = None
    if not args.no_pcg:
        dp.linearize(1)
        dp.damp(lam, False)
        dp.pcg_solve(2, 1e-300)  # warm
        tms = {}
        for n_it in (1, 21):  # tolerance 0 -> exactly n_it iterations
            barrier()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            its, _, _ = dp.pcg_solve(n_it, 1e-300)
            b.record(stream)
            torch.cuda.synchronize()
            tms[n_it] = max_over_ranks(a.elapsed_time(b))
        per_it = (tms[21] - tms[1]) / 20
        pcg = {"ms_per_iteration": per_it, "ms_setup_plus_one_iteration": tms[1],
               "ms_21_iterations": tms[21],
               "note": "RHS + exact Schur block diagonal + its inverse + back-substitution are "
                       "the setup; one iteration = one blocked S'.p term + 3 vector kernels"}

    # ---- stage 2 (RiPoBA) iteration throughput from the lifted state ------------
    stage2 = None
    if not args.no_stage2:
        try:
            s1 = dp.get_state()
            lifted = pv.lift_stage1_to_stage2(s1)
            dp.set_state(lifted)
            f2 = dp.cost(2)
            if math.isfinite(f2):
                lam2 = scfg.initial_lambda

                def it2():
                    nonlocal f2, lam2
                    dp.linearize(2)
                    dp.damp(lam2, True)
                    dp.power_solve(scfg.max_power_order, scfg.power_threshold)
                    ok = dp.trial(2)
                    ft = dp.cost(2, trial=True) if ok else math.inf
                    if ft < f2:
                        dp.accept(2, resolve=False)
                        f2 = ft
                        lam2 = max(scfg.lambda_min, lam2 * scfg.lambda_decrease)
                    else:
                        lam2 = min(scfg.lambda_max, lam2 * scfg.lambda_increase)
                it2()
                barrier()
                torch.cuda.synchronize()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n2 = max(3, args.steps // 2)
                a.record(stream)
                for _ in range(n2):
                    it2()
                b.record(stream)
                torch.cuda.synchronize()
                ms2 = max_over_ranks(a.elapsed_time(b)) / n2
                dp.linearize(2)
                dp.damp(lam2, True)
                kt2 = dp.bench_terms(2, 10)
                stage2 = {"ms_per_iter": ms2, "obs_per_s": n_o / (ms2 * 1e-3),
                          "ms_per_term": max_over_ranks(kt2["term_ms"])}
        except Exception as e:  # report, do not fail the stage-1 line
            stage2 = {"error": f"{type(e).__name__}: {e}"}

    # ---- e2e through the public API: one lm_minimize call of K iterations from a host
    # state in pinned memory to a host result (upload, K iterations, download, trace)
    e2e = None
    if not args.no_e2e:
        cfgK = pv.SolverConfig(max_outer_iterations=args.steps,
                               max_power_order=cfg.max_power_order, function_tolerance=1e-300)
        src = dp.get_state() if stage2 is None else state0
        pin_c = torch.empty(src.cameras.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin_l = torch.empty(src.landmarks.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin_c[...] = src.cameras
        pin_l[...] = src.landmarks
        st_in = pv.ProjectiveState(pin_c, pin_l)
        pv.lm_minimize(problem, st_in, 1, pv.SolverConfig(max_outer_iterations=1), dp=dp)  # warm
        barrier()
        t = time.perf_counter()
        st_out, trace = pv.lm_minimize(problem, st_in, 1, cfgK, dp=dp)
        dt = max_over_ranks(time.perf_counter() - t)
        n_it = len(trace.records) - 1
        bytes_state = st_in.cameras.nbytes + st_in.landmarks.nbytes
        e2e = {"value": n_o * n_it / dt, "unit": "obs/s",
               "h2d_bytes_per_step": bytes_state / n_it,
               "d2h_bytes_per_step": (bytes_state + 8 * n_it) / n_it,
               "ms_per_step": 1e3 * dt / n_it, "steps": n_it,
               "api": "paper_2405_05079_b200.lm_minimize(problem, state, 1, max_outer_iterations=K)",
               "note": "one call: pinned host state upload, K LM iterations, state download"}

    # ---- CPU baseline (rank 0, N=1 only) -----------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, dt, sp = cpu_port_lm(CPU_SAMPLE_FRACTION, iters=2)
        cpu = {"value": v, "unit": "obs/s", "cores": 1, "kind": "port",
               "sample": f"{CPU_SAMPLE_FRACTION:.0%} of vlarge landmarks "
                         f"({sp.num_observations} obs), 2 stage-1 LM iterations, "
                         f"{dt:.2f} s/iter, NumPy oracle port single-threaded"}

    if rank == 0:
        ws = (dp.info()["device_bytes"]) / 1e9
        line = {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (seeded BASELINE vlarge generator, SURVEY App. C)",
                "config": {"workload": f"{args.config} stage-1 PoVar LM iteration",
                           "n_cameras": n_p, "n_landmarks": n_l, "n_obs": n_o,
                           "max_power_order": cfg.max_power_order, "power_threshold": 0.01,
                           "mean_power_order": float(np.mean(orders)) if orders else None,
                           "l2": f"inputs larger than L2 (device working set {ws:.1f} GB)",
                           "parallelism": f"landmark-sharded dp{world}"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(), "spmv": spmv,
                "stage2": stage2, "pcg": pcg}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

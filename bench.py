"""PoVar hot-path benchmark (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[4], the config the metric's target is quoted
on; it fits one B200): the seeded 13,682-camera / 4,456,117-landmark /
~29.0M-observation synthetic problem, fp64, stage-1 PoVar (varpro + power
series, <= 30 terms, threshold 0.01), random N(0,1) start.

* a "step" = one full stage-1 LM iteration (linearize, damp, power series,
  back-substitution, trial, cost, accept + closed-form landmark re-solve).
  ``value`` = n_obs x iterations/s (obs/s) over LM iterations 1..K from the
  random start (north_star's "first 20"), inputs resident in HBM: the W warm-up
  iterations run first and the state is then reset to the start, so ``value``
  and ``e2e`` time the SAME iterations (same power orders, printed for both).
* ``e2e`` = the public ``lm_minimize(max_outer_iterations=K)`` call from a pinned
  host state to a host result (state upload, initial cost, K iterations, state
  download); ``setup_s`` = ``DeviceProblem`` creation (graph sort + upload), the
  one-off cost a first call pays, reported beside it.
* ``spmv`` = the S'.v term alone (the power-series unit of work); ``breakdown``
  = the LM iteration split by operation (CUDA events between the calls).
* ``roofline`` = the dominant term kernel: DRAM-compulsory bytes of the declared
  layout (the L2-resident partials s and vectors t are
  excluded and reported separately) / its time, every block's launch timed with
  CUDA events; ``frac_traffic`` the same with the ncu-measured DRAM bytes.
* ``cpu_baseline`` / ``--impl reference``: the reference's own CPU path (the
  unmodified ``stratba`` installed under baseline/_ref; the NumPy oracle port if
  that install is absent) on a landmark-subsampled slice, at 1 and all host
  threads, with the host recorded.

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


def term_bytes(n_p, n_l, n_o, stage=1, xm_bytes=48):
    """Bytes of one power-series term per kernel group.

    ``dram``: what the declared layout must move between HBM and the SMs per term.
    The camera passes stream the camera-sorted x and m (``xm_bytes``: 32 + 16, or 40 with
    the compact stage-1 stream of PV_OPT_XM) and one int32 id (4) twice -- once for W t, once for W^T v -- plus per camera the 192-byte record
    per pass and y (96); the landmark reduces read each landmark's V+ record (64) and
    (stage 2) its work-slot entry (16) and x (32); the stage-1 reduce reads one 16-byte record
    per 32-landmark slot instead (PV_OPT_KSLOT: L2-resident, not counted).  ``l2``: the transposes that the
    landmark blocking keeps in the persisting L2 by design -- the partials s (written
    and read, 32 per observation) and the vectors t (written per landmark, gathered per
    observation).  ``r1_term``: the reference's own layout (W stored, SURVEY section
    8(d)), for the north_star's roofline figure.
    """
    cam = 2 * (xm_bytes + 4) * n_o + (2 * 192 + 96) * n_p
    lmr = (64 if stage == 1 else 112) * n_l
    l2 = {"cam": 32 * n_o + 32 * n_o, "lm_reduce": 32 * n_o + 32 * n_l}
    r1 = (292 if stage == 1 else 268) * n_o + 52 * n_l + (1632 if stage == 1 else 1408) * n_p
    return {"dram": {"cam": cam, "lm_reduce": lmr}, "l2": l2, "r1_term": r1}


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


def reference_package():
    """The unmodified reference (``stratba``) installed under baseline/_ref, or None."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.exists(os.path.join(path, "stratba", "__init__.py")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    import stratba
    import stratba.solvers  # noqa: F401
    return stratba


def host_record():
    import numpy as np
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")),
                         "")
    except OSError:
        pass
    blas = {}
    try:
        b = np.show_config(mode="dicts")["Build Dependencies"]["blas"]
        blas = {"name": b.get("name"), "version": b.get("version")}
    except Exception:
        pass
    return {"cpu": model, "nproc": len(os.sched_getaffinity(0)), "numpy": np.__version__,
            "blas": blas}


def cpu_lm(fraction, iters, threads, warm=0, seed=0):
    """Time ``iters`` stage-1 LM iterations 1..iters from the random start on a landmark
    subsample of vlarge with ``threads`` BLAS/OpenMP threads: the reference's own
    ``lm_minimize`` (solvers.py:318-393) when installed, else the NumPy oracle port."""
    from threadpoolctl import threadpool_limits

    from paper_2405_05079_b200 import synth
    problem, _ = synth.make_problem(CONFIG, seed, landmark_fraction=fraction)
    state = synth.random_state(problem, 1)
    stratba = reference_package()
    with threadpool_limits(threads):
        if stratba is not None:
            rp = stratba.BaProblem(problem.num_cameras, problem.num_landmarks,
                                   problem.num_observations, problem.camera_indices,
                                   problem.landmark_indices, problem.measurements)
            st = stratba.ProjectiveState(state.cameras, state.landmarks)

            def run(k):
                cfg = stratba.SolverConfig(max_outer_iterations=k, max_power_order=30,
                                           function_tolerance=1e-300)
                t = time.perf_counter()
                _, tr = stratba.solvers.lm_minimize(rp, st, 1, cfg)
                return time.perf_counter() - t, len(tr.records) - 1
            kind = "reference"
        else:
            from oracle import povar_oracle as O
            g = O.graph_of(problem)
            cams, lms = np.array(state.cameras), np.array(state.landmarks)

            def run(k):
                t = time.perf_counter()
                log = O.lm_minimize(g, cams, lms, 1, max_iterations=k, max_order=30,
                                    ftol=1e-300)
                return time.perf_counter() - t, len(log.decisions)
            kind = "port"
        if warm:
            run(warm)
        dt, n_it = run(iters)
    return {"obs_per_s": problem.num_observations * n_it / dt, "s_per_iter": dt / n_it,
            "iterations": n_it, "threads": threads, "kind": kind,
            "n_obs": problem.num_observations}, problem


def run_reference(args, rank, world):
    if rank != 0:
        return
    fr = CPU_SAMPLE_FRACTION
    nthr = len(os.sched_getaffinity(0))
    r, problem = cpu_lm(fr, args.steps, nthr, warm=max(1, args.warmup))
    value = r["obs_per_s"]
    what = ("stratba.lm_minimize (baseline/_ref, unmodified reference)" if r["kind"] == "reference"
            else "NumPy oracle port (oracle/povar_oracle.py)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "obs/s",
            "n_gpus": world, "steps": r["iterations"], "warmup": args.warmup,
            "ms_per_step": 1e3 * r["s_per_iter"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE vlarge generator, landmark-subsampled)",
            "config": {"workload": f"vlarge stage-1 PoVar LM iterations 1..K, {what}",
                       "landmark_fraction": fr, "n_cameras": problem.num_cameras,
                       "n_landmarks": problem.num_landmarks,
                       "n_obs": problem.num_observations, "max_power_order": 30},
            "cpu_baseline": {"value": value, "unit": "obs/s", "cores": nthr, "kind": r["kind"],
                             "sample": f"{fr:.0%} of vlarge landmarks "
                                       f"({problem.num_observations} obs), LM iterations "
                                       f"1..{r['iterations']} from the random start, {what}",
                             "host": host_record()},
            "e2e": {"value": value, "unit": "obs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
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
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    dp = pv.DeviceProblem(problem, 0.1, device=local, rank=rank, world=world, nccl_id=nccl_id,
                          lm_range=plan[rank])
    setup_s = time.perf_counter() - t_setup
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

    def ev():
        e = torch.cuda.Event(enable_timing=True)
        e.record(stream)
        return e

    # ---- LM iterations 1..K from the random start (value) --------------------------
    run = {}
    ops = ("linearize", "damp", "power_solve", "trial_cost", "accept_resolve")

    def start_run():
        dp.set_state(state0)
        run.update(f=dp.cost(1), lam=scfg.initial_lambda, linearized=False, orders=[],
                   marks=[], solve={})

    def lm_iteration(timed=False):
        # solver.lm_minimize's iteration: a rejected step leaves the state unchanged, so its
        # linearization (and, POSE_ONLY, the reduced RHS) is reused
        m = [ev()] if timed else None
        if not run["linearized"]:
            dp.linearize(1)
            run["linearized"] = True
        if timed:
            m.append(ev())
        dp.damp(run["lam"], False)
        if timed:
            m.append(ev())
        order, _ = dp.power_solve(scfg.max_power_order, scfg.power_threshold)
        run["orders"].append(order)
        if timed:
            m.append(ev())
            inf = dp.info()
            for k in ("solve_rhs_us", "solve_terms_us", "solve_backsub_us",
                      "solve_terms_launched"):
                run["solve"][k] = run["solve"].get(k, 0) + inf[k]
        ok = dp.trial(1)
        ft = dp.cost(1, trial=True) if ok else math.inf
        if timed:
            m.append(ev())
        if ft < run["f"]:
            run["f"], _ = dp.accept(1, resolve=True)
            run["linearized"] = False
            run["lam"] = max(scfg.lambda_min, run["lam"] * scfg.lambda_decrease)
        else:
            run["lam"] = min(scfg.lambda_max, run["lam"] * scfg.lambda_increase)
        if timed:
            m.append(ev())
            run["marks"].append(m)

    start_run()
    for _ in range(args.warmup):
        lm_iteration()
    start_run()  # iterations 1..K, exactly those e2e times
    launches0 = dp.info()["launches"]
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        e0 = ev()
        for _ in range(args.steps):
            lm_iteration(timed=True)
        e1 = ev()
        torch.cuda.synchronize()
    barrier()
    ms_total = max_over_ranks(e0.elapsed_time(e1))
    launches = dp.info()["launches"] - launches0
    ms_step = ms_total / args.steps
    value = n_o * args.steps / (ms_total * 1e-3)
    orders = list(run["orders"])
    accepts = []
    breakdown = {k: 0.0 for k in ops}
    for m in run["marks"]:
        for k, a, b in zip(ops, m, m[1:]):
            breakdown[k] += a.elapsed_time(b) / args.steps
    breakdown = {k: round(max_over_ranks(v), 4) for k, v in breakdown.items()}
    # the power solve split (device time inside pv_power_solve, povar.cu op_power)
    breakdown.update({
        "solve_rhs": round(run["solve"]["solve_rhs_us"] / 1e3 / args.steps, 4),
        "solve_terms": round(run["solve"]["solve_terms_us"] / 1e3 / args.steps, 4),
        "solve_backsub": round(run["solve"]["solve_backsub_us"] / 1e3 / args.steps, 4),
        "terms_launched_per_step": run["solve"]["solve_terms_launched"] / args.steps})

    # ---- S'.v terms and per-kernel roofline (at the state after iteration K) ---------
    dp.linearize(1)
    dp.damp(run["lam"], False)
    dp.power_solve(1, 0.0)
    dp.bench_terms(1, 3)
    barrier()
    kt = dp.bench_terms(1, 20)
    kt = {k: max_over_ranks(v) for k, v in kt.items()}
    peak, peak_src = _peaks()
    loc = dp.info()
    # one warp per camera: the persistent TMA-pipelined camera kernel runs the blocks
    cam_name = "k_cam_pipe" if loc["warps_per_cam"] == 1 else "k_cam"

    def term_report(kt, stage):
        tb = term_bytes(n_p, loc["n_l_local"], loc["n_o_local"], stage,
                        xm_bytes=loc["xm_bytes"] if stage == 1 else 48)
        kern = {}
        for name, key, tkey in (("k_lm_reduce", "lm_reduce", "lm_reduce_ms"),
                                (cam_name, "cam", "cam_ms")):
            ms = kt[tkey]
            gbs = tb["dram"][key] / (ms * 1e-3) / 1e9
            kern[name] = {"ms": ms, "dram_bytes": tb["dram"][key], "l2_bytes": tb["l2"][key],
                          "achieved_gbs": gbs, "frac": gbs / peak}
        term_ms = kt["term_ms"]
        dram = sum(tb["dram"].values())
        return {"ms_per_term": term_ms, "terms_per_s": 1e3 / term_ms,
                "obs_per_s": n_o / (term_ms * 1e-3),
                "dram_bytes_per_term": dram,
                "dram_frac": dram / (term_ms * 1e-3) / 1e9 / peak,
                "r1_equivalent_gbs": tb["r1_term"] * world / (term_ms * 1e-3) / 1e9,
                "r1_equivalent_frac_of_8tbs": tb["r1_term"] * world / (term_ms * 1e-3) / 8e12,
                "kernels": kern, "blocks": int(kt["blocks"])}

    spmv = term_report(kt, 1)
    kern = spmv["kernels"]
    dom = max(kern, key=lambda k: kern[k]["ms"])
    traffic = traffic_from_profile(dom, n_o)
    roofline = {"bound": "hbm", "achieved": kern[dom]["achieved_gbs"], "peak": peak,
                "unit": "GB/s", "frac": kern[dom]["frac"], "traffic": traffic,
                "frac_traffic": (traffic / (kern[dom]["ms"] * 1e-3) / 1e9 / peak
                                 if traffic else None),
                "kernel": dom, "peak_source": peak_src,
                "note": "per power-series term, summed over the landmark-block launches: "
                        "achieved = DRAM-compulsory bytes of the layout / summed launch time "
                        "(CUDA events around every launch); traffic = ncu dram bytes"}
    # the series' own device time (events around the term graph inside pv_power_solve): the
    # terms actually launched per solve (order + 1: the term that takes the stop is applied,
    # solvers.py:140-149) and what one of them takes inside the graph
    tl = breakdown["terms_launched_per_step"]
    ms_term_series = breakdown["solve_terms"] / tl if tl else None
    non_term_ms = ms_step - breakdown["solve_terms"]

    # ---- PCG inner solver ("iterative", solvers.py:153-187) on the same system -----
    pcg = None
    if not args.no_pcg:
        dp.linearize(1)
        dp.damp(run["lam"], False)
        dp.pcg_solve(2, 1e-300)  # warm
        tms = {}
        for n_it in (1, 21):  # tolerance 0 -> exactly n_it iterations
            barrier()
            torch.cuda.synchronize()
            a = ev()
            dp.pcg_solve(n_it, 1e-300)
            b = ev()
            torch.cuda.synchronize()
            tms[n_it] = max_over_ranks(a.elapsed_time(b))
        pcg = {"ms_per_iteration": (tms[21] - tms[1]) / 20,
               "ms_setup_plus_one_iteration": tms[1], "ms_21_iterations": tms[21],
               "note": "RHS + exact Schur block diagonal + its inverse + back-substitution are "
                       "the setup; one iteration = one blocked S'.p term + 3 vector kernels"}

    # ---- stage 2 (RiPoBA) iteration throughput from the lifted state ------------
    stage2 = None
    if not args.no_stage2:
        try:
            s1 = dp.get_state()
            lifted = pv.lift_stage1_to_stage2(s1)
            dp.set_state(lifted)
            st2 = {"f": dp.cost(2), "lam": scfg.initial_lambda, "orders": []}
            if math.isfinite(st2["f"]):
                def it2():
                    dp.linearize(2)
                    dp.damp(st2["lam"], True)
                    o, _ = dp.power_solve(scfg.max_power_order, scfg.power_threshold)
                    st2["orders"].append(o)
                    ok = dp.trial(2)
                    ft = dp.cost(2, trial=True) if ok else math.inf
                    if ft < st2["f"]:
                        dp.accept(2, resolve=False)
                        st2["f"] = ft
                        st2["lam"] = max(scfg.lambda_min, st2["lam"] * scfg.lambda_decrease)
                    else:
                        st2["lam"] = min(scfg.lambda_max, st2["lam"] * scfg.lambda_increase)
                it2()
                st2["orders"].clear()
                barrier()
                torch.cuda.synchronize()
                n2 = max(3, args.steps // 2)
                a = ev()
                for _ in range(n2):
                    it2()
                b = ev()
                torch.cuda.synchronize()
                ms2 = max_over_ranks(a.elapsed_time(b)) / n2
                dp.linearize(2)
                dp.damp(st2["lam"], True)
                kt2 = {k: max_over_ranks(v) for k, v in dp.bench_terms(2, 10).items()}
                t2 = term_report(kt2, 2)
                k2 = t2["kernels"]
                d2 = max(k2, key=lambda k: k2[k]["ms"])
                stage2 = {"ms_per_iter": ms2, "obs_per_s": n_o / (ms2 * 1e-3), "iterations": n2,
                          "mean_power_order": float(np.mean(st2["orders"])),
                          "ms_per_term": t2["ms_per_term"], "spmv": t2,
                          "roofline": {"bound": "hbm", "kernel": d2,
                                       "achieved": k2[d2]["achieved_gbs"], "peak": peak,
                                       "unit": "GB/s", "frac": k2[d2]["frac"]}}
        except Exception as e:  # report, do not fail the stage-1 line
            stage2 = {"error": f"{type(e).__name__}: {e}"}

    # ---- e2e through the public API: one lm_minimize call of K iterations from the
    # random start in pinned host memory to a host result -- the iterations value timed
    e2e = None
    if not args.no_e2e:
        cfgK = pv.SolverConfig(max_outer_iterations=args.steps,
                               max_power_order=cfg.max_power_order, function_tolerance=1e-300)
        pin_c = torch.empty(state0.cameras.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin_l = torch.empty(state0.landmarks.shape, dtype=torch.float64, pin_memory=True).numpy()
        pin_c[...] = state0.cameras
        pin_l[...] = state0.landmarks
        st_in = pv.ProjectiveState(pin_c, pin_l)
        pv.lm_minimize(problem, st_in, 1, pv.SolverConfig(max_outer_iterations=1), dp=dp)  # warm
        barrier()
        decisions = []
        t = time.perf_counter()
        st_out, trace = pv.lm_minimize(problem, st_in, 1, cfgK, dp=dp, decisions=decisions)
        dt = max_over_ranks(time.perf_counter() - t)
        n_it = len(trace.records) - 1
        e_orders = [d["order"] for d in decisions]
        bytes_state = st_in.cameras.nbytes + st_in.landmarks.nbytes
        e2e = {"value": n_o * n_it / dt, "unit": "obs/s",
               "h2d_bytes_per_step": bytes_state / n_it,
               "d2h_bytes_per_step": (bytes_state + 8 * (n_it + 1)) / n_it,
               "ms_per_step": 1e3 * dt / n_it, "steps": n_it,
               "mean_power_order": float(np.mean(e_orders)),
               "same_iterations_as_value": e_orders == orders,
               "setup_s": max_over_ranks(setup_s),
               "value_incl_setup": n_o * n_it / (dt + max_over_ranks(setup_s)),
               "api": "paper_2405_05079_b200.lm_minimize(problem, state, 1, "
                      "max_outer_iterations=K)",
               "note": "one call: pinned host state upload, initial cost, LM iterations 1..K "
                       "from the random start, state download; setup_s = DeviceProblem "
                       "creation (graph sort, work lists, upload), paid once per problem"}

    # ---- CPU baseline (rank 0, N=1 only): the reference at 1 and all host threads -----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nthr = len(os.sched_getaffinity(0))
        runs = [cpu_lm(CPU_SAMPLE_FRACTION, 2, t, warm=1 if t == 1 else 0)[0]
                for t in sorted({1, nthr})]
        best = max(runs, key=lambda r: r["obs_per_s"])
        cpu = {"value": best["obs_per_s"], "unit": "obs/s", "cores": best["threads"],
               "kind": best["kind"],
               "sample": f"{CPU_SAMPLE_FRACTION:.0%} of vlarge landmarks ({best['n_obs']} obs), "
                         f"LM iterations 1..2 from the random start, "
                         + ("stratba.lm_minimize (baseline/_ref)" if best["kind"] == "reference"
                            else "NumPy oracle port"),
               "by_threads": {str(r["threads"]): r["obs_per_s"] for r in runs},
               "host": host_record()}

    if rank == 0:
        ws = (dp.info()["device_bytes"]) / 1e9
        line = {"metric": METRIC, "value": value, "unit": "obs/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
                "dtype": "f64",
                "data": "synthetic (seeded BASELINE vlarge generator, SURVEY App. C)",
                "config": {"workload": f"{args.config} stage-1 PoVar LM iterations 1..K from "
                                       "the random N(0,1) start",
                           "n_cameras": n_p, "n_landmarks": n_l, "n_obs": n_o,
                           "max_power_order": cfg.max_power_order, "power_threshold": 0.01,
                           "mean_power_order": float(np.mean(orders)) if orders else None,
                           "power_orders": orders,
                           "l2": f"inputs larger than L2 (device working set {ws:.1f} GB)",
                           "parallelism": f"landmark-sharded dp{world}"},
                "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": launches, "clocks": clk.summary(),
                "ms_per_term": spmv["ms_per_term"], "ms_per_term_in_series": ms_term_series,
                "non_term_ms_per_step": non_term_ms,
                "breakdown_ms_per_step": breakdown, "setup_s": setup_s, "spmv": spmv,
                "stage2": stage2, "pcg": pcg}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

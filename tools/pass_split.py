"""Time the two camera passes on their own (PV_OPT_BENCH_SPLIT) for each camera kernel.
Usage: python tools/pass_split.py [config] [stage] [versions, e.g. 1,2]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
versions = [int(v) for v in (sys.argv[3] if len(sys.argv) > 3 else "1,2").split(",")]
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
n_o = problem.num_observations
for rnd in range(2):
    for v in versions:
        dp.set_option(_lib.PV_OPT_CAM_PIPE, v)
        dp.linearize(stage)
        dp.damp(1e-4, stage == 2)
        dp.power_solve(1, 0.0)
        dp.set_option(_lib.PV_OPT_BENCH_SPLIT, 1)
        dp.bench_terms(stage, 2)
        r = dp.bench_terms(stage, 5)
        dp.set_option(_lib.PV_OPT_BENCH_SPLIT, 0)
        t = dp.bench_terms(stage, 5)
        ha, hc = r["lm_reduce_ms"], r["cam_ms"]
        print(f"round {rnd} pipe v{v}: W^T v pass {ha:.4f} ms ({n_o * 52 / ha / 1e9:.0f} GB/s "
              f"stream), W t pass {hc:.4f} ms ({n_o * 52 / hc / 1e9:.0f} GB/s stream); fused term "
              f"{t['term_ms']:.4f} ms (cam {t['cam_ms']:.4f}, reduce {t['lm_reduce_ms']:.4f})",
              flush=True)

"""Where a term of the series kernel spends its time (diagnostic build -DPV_SER_TIMING,
tools/build_variants.sh "stime:-DPV_SER_TIMING"): CTA 0's time between grid barriers (every
step of one term) and, for one step, every warp's R / ring split and finish-time spread.
Usage: PV_LIB_PATH=build_ab/libpovar_stime.so python tools/series_times.py [config] [step] [stage]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
step = int(sys.argv[2]) if len(sys.argv) > 2 else 5
stage = int(sys.argv[3]) if len(sys.argv) > 3 else 1
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
st = synth.random_state(problem, 1)
if stage == 2:
    st = pv.lift_stage1_to_stage2(st)
dp.set_state(st)
dp.linearize(stage)
dp.damp(1e-4, stage == 2)
for kv in sys.argv[4:]:
    k, v = kv.split("=")
    dp.set_option(getattr(_lib, k), int(v))
fn = dp._lib.pv_debug_series_times
fn.restype = ctypes.c_int
B = dp.info()["blocks"]
W = dp.info()["pipe_warps"]
fn(dp._ctx, ctypes.c_int(2), ctypes.c_int(step), None, None, None, None)
dp.bench_terms(stage, 3)
r = dp.bench_terms(stage, 10)
bar = np.zeros(64, np.uint64)
wt = np.zeros(3 * W, np.uint64)
assert fn(dp._ctx, ctypes.c_int(2), ctypes.c_int(step), bar.ctypes.data_as(ctypes.c_void_p),
          wt.ctypes.data_as(ctypes.c_void_p), None, None) == 0
bar = bar.astype(np.int64)
d = np.diff(bar[:B + 4]) / 1e3
print(f"term {r['term_ms'] * 1e3:.1f} us; CTA 0 between barriers (us): steps -2..{B - 1}: "
      + " ".join(f"{x:.1f}" for x in d[:B + 2]) + f" | epilogue+decision {d[B + 2]:.1f}; sum {d.sum():.1f}")
wt = wt.reshape(W, 3).astype(np.int64)
t0 = wt[:, 0].min()
s, r_end, e = (wt[:, 0] - t0) / 1e3, (wt[:, 1] - t0) / 1e3, (wt[:, 2] - t0) / 1e3
print(f"step {step}: start spread {s.max():.1f}; R phase per warp: mean {np.mean(r_end - s):.1f} "
      f"p99 {np.percentile(r_end - s, 99):.1f} max {np.max(r_end - s):.1f}; ring: mean {np.mean(e - r_end):.1f} "
      f"max {np.max(e - r_end):.1f}; finish: min {e.min():.1f} p10 {np.percentile(e, 10):.1f} median "
      f"{np.median(e):.1f} p90 {np.percentile(e, 90):.1f} p99 {np.percentile(e, 99):.1f} max {e.max():.1f} us")

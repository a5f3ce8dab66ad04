"""Per-warp timers of one fused launch of the persistent camera kernel (diagnostic build
-DPV_PIPE_TIMING, tools/build_variants.sh "timing:-DPV_PIPE_TIMING"): finish-time spread,
and a least-squares fit of a warp's duration on its work (items, 32-observation rounds,
observations, cameras finished) -- the cost model of the work-list balance (PV_OPT_BAL_*).
Usage: PV_LIB_PATH=build_ab/libpovar_timing.so python tools/pipe_times.py [config] [block] [mode:item:round:last]"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
blk = int(sys.argv[2]) if len(sys.argv) > 2 else 5
combo = sys.argv[3] if len(sys.argv) > 3 else "1:24:0:0"
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(1)
dp.damp(1e-4, False)
mode, item, rnd, last = (int(x) for x in combo.split(":"))
dp.set_option(_lib.PV_OPT_BAL_ITEM, item)
dp.set_option(_lib.PV_OPT_BAL_ROUND, rnd)
dp.set_option(_lib.PV_OPT_BAL_LAST, last)
dp.set_option(_lib.PV_OPT_BALANCE, mode)
lib = dp._lib
fn = lib.pv_debug_pipe_times
fn.restype = ctypes.c_int
B = dp.info()["blocks"]
n_items = ctypes.c_int(0)
fn(dp._ctx, ctypes.c_int(blk), None, ctypes.byref(n_items), None, ctypes.c_int(0), None)
dp.bench_terms(1, 3)
W = dp.info()["pipe_warps"]
# find W from the offsets: 3 * B * (W + 1) ints
items = np.zeros((n_items.value, 4), np.int32)
for Wt in (W, 148 * 4 * 3, 148 * 6 * 3, 148 * 3 * 3):
    pass
off = np.zeros(3 * B * (W + 1), np.int32)
t = np.zeros(3 * W, np.uint64)
rc = fn(dp._ctx, ctypes.c_int(blk), t.ctypes.data_as(ctypes.c_void_p), ctypes.byref(n_items),
        items.ctypes.data_as(ctypes.c_void_p), ctypes.c_int(len(items)),
        off.ctypes.data_as(ctypes.c_void_p))
assert rc == 0
t = t.reshape(W, 3).astype(np.int64)
t0 = t[:, 0].min()
start, end, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, t[:, 2]
dur = end - start
print(f"launch of block {blk}: warps {W}, start spread {start.max():.1f} us, end: min {end.min():.1f} "
      f"p10 {np.percentile(end, 10):.1f} median {np.median(end):.1f} p90 {np.percentile(end, 90):.1f} "
      f"p99 {np.percentile(end, 99):.1f} max {end.max():.1f} us")
off = off.reshape(3, B, W + 1)
feat = np.zeros((W, 5))
for w in range(W):
    for L, b in ((0, blk), (2, blk + 1)):
        it = items[off[L, b, w]:off[L, b, w + 1]]
        n = it[:, 2]
        feat[w, 0] += len(it)
        feat[w, 1] += ((n + 31) // 32).sum()
        feat[w, 2] += n.sum()
        if L == 0:
            feat[w, 3] += ((it[:, 3] & 2) != 0).sum()
    feat[w, 4] = 1.0
coef, *_ = np.linalg.lstsq(feat, dur, rcond=None)
pred = feat @ coef
print("fit dur_us = %.4f*items + %.4f*rounds + %.5f*obs + %.4f*cams + %.2f ; residual rms %.2f us "
      "(dur rms about mean %.2f us)" % (*coef, np.sqrt(np.mean((dur - pred) ** 2)), dur.std()))
print("in observation-equivalents: item %.1f round %.1f last %.1f" %
      (coef[0] / coef[2], coef[1] / coef[2], coef[3] / coef[2]))
# per-SM effects: mean residual by SM
res = dur - pred
bysm = np.array([res[sm == s].mean() for s in np.unique(sm)])
print(f"residual by SM: std {bysm.std():.2f} us, min {bysm.min():.2f}, max {bysm.max():.2f}; "
      f"per-warp features: items {feat[:, 0].mean():.1f} obs {feat[:, 2].mean():.0f}")
np.save(os.path.join(ROOT, "gpurun_out", "pipe_times.npy"), np.column_stack([start, end, sm, feat]))

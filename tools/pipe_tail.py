"""Per-consumer-warp start/end times of one k_cam_pipe2 launch (diagnostic build with
-DPV_PIPE2_TIMING): how long the persistent grid's tail is.
Usage: PV_LIB_PATH=build_ab/libpovar_timing.so python tools/pipe_tail.py [config]"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_option(_lib.PV_OPT_CAM_PIPE, 2)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(1)
dp.damp(1e-4, False)
dp.bench_terms(1, 2)
lib = _lib.load()
t = np.zeros(2 * 8192, dtype=np.uint64)
items = np.zeros(8192, dtype=np.int32)
n = ctypes.c_int()
fn = lib.pv_debug_pipe2_times
entry = np.zeros(4096, dtype=np.uint64)
fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int),
               ctypes.c_void_p]
_lib.check(fn(dp._ctx, t.ctypes.data, items.ctypes.data, ctypes.byref(n), entry.ctypes.data),
           dp._ctx)
W = n.value
st, en = t[0:2 * W:2].astype(np.float64), t[1:2 * W:2].astype(np.float64)
ent = entry[:W // 3].astype(np.float64)
t0 = ent.min()
print(f"CTA entry spread {(ent.max() - t0) / 1e3:.1f} us; consumers start "
      f"{(st.min() - t0) / 1e3:.1f}..{(st.max() - t0) / 1e3:.1f} us after the first CTA entry")
st, en = (st - t0) / 1e3, (en - t0) / 1e3
dur = en - st
print(f"{W} consumer warps; start spread {st.max():.1f} us; end: min {en.min():.1f} "
      f"median {np.median(en):.1f} p90 {np.percentile(en, 90):.1f} max {en.max():.1f} us; "
      f"items/warp mean {items[:W].mean():.1f} max {items[:W].max()}")
print("busy fraction of the launch (sum of warp durations / (W x max end)):",
      round(dur.sum() / (W * en.max()), 3))
order = np.argsort(en)[-10:]
print("slowest warps (end us, items):", [(round(en[i], 1), int(items[i])) for i in order])

import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import _lib
from _pvutil import golden, problem_from
z = golden("tiny_lm.npz")
what = sys.argv[1]
st = pv.ProjectiveState(z["s2_cams0"], z["s2_lms0"])
dp = pv.DeviceProblem(problem_from(z), 0.1)
dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
dp.set_state(st); dp.linearize(2); dp.damp(1e-4, True)
try:
    if what.startswith("bench"):
        print(what, "ok", dp.bench_terms(2, int(what[5:])))
    else:
        print(what, "ok", dp.power_solve(int(what[5:]), 0.0))
except Exception as e:
    print(what, "FAIL", str(e)[-60:])
    import ctypes
    out=(ctypes.c_int64*24)(); dp._lib.pv_info(dp._ctx, out); print("marker", out[23])

import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import _lib
from _pvutil import golden, problem_from
z = golden("tiny_lm.npz")
st = pv.ProjectiveState(z["cams"], z["lms"])
for blk in (64 << 10, 1 << 30):
  for order in (1, 2, 5):
    res = []
    for series in (0, 1):
        dp = pv.DeviceProblem(problem_from(z), 0.1)
        dp.set_option(_lib.PV_OPT_BLOCK_BYTES, blk)
        dp.set_option(_lib.PV_OPT_SERIES, series)
        dp.set_state(st); dp.linearize(1); dp.damp(1e-4, False)
        o, tr = dp.power_solve(order, 0.0)
        res.append((o, tr, dp.debug(_lib.PV_DBG_X).copy()))
    d = np.abs(res[0][2] - res[1][2]).max()
    print("blocks", dp.info()["blocks"], "order", order, res[0][0], res[1][0], "trunc", res[0][1], res[1][1], "max|dx diff|", d, flush=True)

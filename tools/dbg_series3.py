import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import _lib
from _pvutil import golden, problem_from
z = golden("tiny_lm.npz")
tag = os.environ.get("PV_LIB_PATH", "default")
for stage, xm in ((1, 1), (1, 0), (2, 0)):
    st = pv.ProjectiveState(z["cams"], z["lms"]) if stage == 1 else pv.ProjectiveState(z["s2_cams0"], z["s2_lms0"])
    res = []
    try:
        for series in (0, 1):
            dp = pv.DeviceProblem(problem_from(z), 0.1)
            dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
            dp.set_option(_lib.PV_OPT_SERIES, series)
            dp.set_option(_lib.PV_OPT_XM, xm)
            dp.set_state(st); dp.linearize(stage); dp.damp(1e-4, stage == 2)
            o, tr = dp.power_solve(20, 0.01)
            res.append((o, dp.debug(_lib.PV_DBG_X).copy()))
        print(tag, "stage", stage, "xm", xm, "orders", res[0][0], res[1][0], "max diff", np.abs(res[0][1] - res[1][1]).max(), flush=True)
    except Exception as e:
        print(tag, "stage", stage, "xm", xm, "FAIL", str(e)[-50:], flush=True)
        break

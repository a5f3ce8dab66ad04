import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import _lib
from _pvutil import golden, problem_from
z = golden("tiny_lm.npz")
st = pv.ProjectiveState(z["cams"], z["lms"])
for name, knobs in (("pipe graph", []), ("pipe hostloop", [(_lib.PV_OPT_GRAPH, 0)]), ("xm0", [(_lib.PV_OPT_XM, 0)]),
                    ("series", [(_lib.PV_OPT_SERIES, 1)]), ("bal0", [(_lib.PV_OPT_BALANCE, 0)])):
    try:
        dp = pv.DeviceProblem(problem_from(z), 0.1)
        dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
        for k, v in knobs:
            dp.set_option(k, v)
        dp.set_state(st); dp.linearize(1); dp.damp(1e-4, False)
        print(name, "ok", dp.power_solve(20, 0.01), flush=True)
    except Exception as e:
        print(name, "FAIL", str(e)[-70:], flush=True)
        break

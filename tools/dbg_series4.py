import sys, os, ctypes
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import _lib
from _pvutil import golden, problem_from
z = golden("tiny_lm.npz")
st = pv.ProjectiveState(z["cams"], z["lms"])
def get(dp, which, n):
    out = np.zeros(n)
    dp._call("pv_debug_get", which, _lib.dptr(out))
    return out
for order in (1, 2):
    res = []
    for series in (0, 1):
        dp = pv.DeviceProblem(problem_from(z), 0.1)
        dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
        dp.set_option(_lib.PV_OPT_SERIES, series)
        dp.set_option(_lib.PV_OPT_XM, 0)
        dp.set_option(_lib.PV_OPT_GRAPH, 0)
        dp.set_state(st); dp.linearize(1); dp.damp(1e-4, False)
        o, tr = dp.power_solve(order, 0.0)
        res.append((o, tr, dp.debug(_lib.PV_DBG_X).copy(), get(dp, 100, dp.n_p * 12), get(dp, 101, dp.n_p * 12), get(dp, 102, dp.n_l_local * 4)))
    a, b = res
    print("order", order, "trunc", a[1], b[1])
    for name, i in (("x", 2), ("y", 3), ("v", 4), ("t", 5)):
        d = np.abs(a[i] - b[i]).reshape(-1)
        print("  ", name, "max diff", d.max(), "n bad", int((d > 1e-9 * (1 + np.abs(a[i].reshape(-1)))).sum()), "of", d.size, "first bad", int(np.argmax(d > 0)) if d.max() > 0 else -1)
    bad = np.abs(a[3] - b[3]).reshape(-1, 12).max(axis=1)
    print("   bad cameras (y):", np.nonzero(bad > 1e-9)[0][:20])
    badt = np.abs(a[5] - b[5]).reshape(-1, 4).max(axis=1)
    print("   bad landmarks (t):", np.nonzero(badt > 1e-9)[0][:20], int((badt > 1e-9).sum()))
    ta, tb = a[5].reshape(-1, 4), b[5].reshape(-1, 4)
    for l in (0, 1, 2, 1000):
        print("   lm", l, "ref", ta[l], "series", tb[l])
    print("   bad components per column:", (np.abs(ta - tb) > 1e-9 * (1 + np.abs(ta))).sum(axis=0))

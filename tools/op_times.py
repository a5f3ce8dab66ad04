"""Per-operation wall times of stage-1 LM iterations through the DeviceProblem API
(each op synchronises the stream).  Usage: python tools/op_times.py [config] [iters]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
problem, _ = synth.make_problem(name, 0)
state = synth.random_state(problem, 1)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(state)
f = dp.cost(1)
lam = 1e-4
tim = {}


def t(key, fn, *a):
    t0 = time.perf_counter()
    out = fn(*a)
    tim.setdefault(key, []).append((time.perf_counter() - t0) * 1e3)
    return out


for it in range(iters):
    t("linearize", dp.linearize, 1)
    t("damp", dp.damp, lam, False)
    order, _ = t("power", dp.power_solve, synth.CONFIGS[name].max_power_order, 0.01)
    tim.setdefault("order", []).append(order)
    t("trial", dp.trial, 1)
    ft = t("cost_trial", dp.cost, 1, True)
    if ft < f:
        f, _ = t("accept_resolve", dp.accept, 1, True)
        lam *= 0.5
    else:
        lam *= 4
for k, v in tim.items():
    v = np.array(v[1:] if len(v) > 1 else v)
    print(f"{k:16s} mean {v.mean():8.3f}  min {v.min():8.3f}  (n={len(v)})")

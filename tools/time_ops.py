"""Wall time of individual DeviceProblem operations (each synchronises) on a BASELINE config.
Usage: [PV_LIB_PATH=...] python tools/time_ops.py [config] [reps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
ops = {
    "linearize1": lambda: dp.linearize(1),
    "damp": lambda: dp.damp(1e-4, False),
    "power(30, 0)": lambda: dp.power_solve(30, 0.0),
    "trial": lambda: dp.trial(1),
    "cost_trial": lambda: dp.cost(1, trial=True),
    "resolve_current": lambda: dp.resolve_current(),
}
res = {}
for _ in range(reps):
    for k, fn in ops.items():
        t0 = time.perf_counter()
        fn()
        res.setdefault(k, []).append((time.perf_counter() - t0) * 1e3)
tag = os.environ.get("PV_LIB_PATH", "default")
for k, v in res.items():
    v = np.array(v[1:])
    print(f"{tag} {k:16s} median {np.median(v):8.3f} ms  min {v.min():8.3f}")

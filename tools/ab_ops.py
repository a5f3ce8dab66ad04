"""A/B pv_set_option knobs on whole operations (power solve, PCG, LM iteration) at a config.
Usage: AB="9=0|9=1" ROUNDS=3 python tools/ab_ops.py [config]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
variants = [[tuple(int(x) for x in kv.split("=")) for kv in v.split(",") if kv]
            for v in os.environ.get("AB", "9=0|9=1").split("|")]
rounds = int(os.environ.get("ROUNDS", "3"))
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(1)
dp.damp(1e-4, False)
res = {}
ref = None
for rnd in range(rounds):
    for i, var in enumerate(variants):
        for k, v in var:
            dp.set_option(k, v)
        t0 = time.perf_counter()
        order, _ = dp.power_solve(30, 0.0)
        t1 = time.perf_counter()
        dx = dp.step(1)[0].copy()
        its, _, _ = dp.pcg_solve(20, 1e-300)
        t2 = time.perf_counter()
        if ref is None:
            ref = dx
        assert np.array_equal(dx, ref), (i, float(np.abs(dx - ref).max()))
        res.setdefault(i, []).append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
for i, var in enumerate(variants):
    a = np.array(res[i][1:] if rounds > 1 else res[i])
    print(f"variant {i} {var}: power(30 terms) {np.median(a[:, 0]):.3f} ms  "
          f"pcg(20 its) {np.median(a[:, 1]):.3f} ms  (bit-identical steps)")

"""Time one power-series term (pv_bench_terms) on a BASELINE config; PV_LIB_PATH picks a build.
Usage: [PV_LIB_PATH=...] python tools/time_terms.py [config]"""
import os, sys
sys.path.insert(0, os.getcwd())
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import synth
problem, _ = synth.make_problem(sys.argv[1], 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(1); dp.damp(1e-4, False)
dp.bench_terms(1, 3)
for _ in range(2):
    r = dp.bench_terms(1, 10); print(os.environ.get("PV_LIB_PATH"), {k: round(v, 4) for k, v in r.items()})

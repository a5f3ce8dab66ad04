"""Set up a linearized, damped system on a BASELINE config and run power-series
terms through pv_bench_terms (no stop test), for ncu captures of the term kernels.
Usage: python tools/profile_terms.py [config] [stage] [terms] [key=value,...]
(the optional last argument sets pv_set_option knobs first, e.g. 8=1)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
terms = int(sys.argv[3]) if len(sys.argv) > 3 else 2
knobs = [tuple(int(x) for x in kv.split("=")) for kv in sys.argv[4].split(",")] \
    if len(sys.argv) > 4 else []
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
for k, v in knobs:
    dp.set_option(k, v)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(stage)
dp.damp(1e-4, stage == 2)
print(dp.bench_terms(stage, terms))

"""Run the landmark re-solve (k_resolve_slots) a few times on a BASELINE config (ncu target).
Usage: python tools/profile_resolve.py [config] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
st = synth.random_state(problem, 1)
for _ in range(reps):
    dp.set_state(st)
    print("rank-deficient", dp.resolve_current())

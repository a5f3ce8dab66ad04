"""Run a few stage-1 LM iterations on a BASELINE config (for ncu launch lists /
captures).  Usage: python tools/profile_step.py [config] [iters] [stage2]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 4
cfg = synth.CONFIGS[cfg_name]
problem, _ = synth.make_problem(cfg_name, 0)
state = synth.random_state(problem, 1)
dp = pv.DeviceProblem(problem, 0.1)
scfg = pv.SolverConfig(max_outer_iterations=iters, max_power_order=cfg.max_power_order,
                       function_tolerance=1e-300)
final, trace = pv.lm_minimize(problem, state, 1, scfg, dp=dp)
print("stage1 costs", [r.cost for r in trace.records])
if len(sys.argv) > 3:
    lifted = pv.lift_stage1_to_stage2(final)
    f2, tr2 = pv.lm_minimize(problem, lifted, 2, pv.SolverConfig(max_outer_iterations=2,
                             max_power_order=cfg.max_power_order), dp=dp)
    print("stage2 costs", [r.cost for r in tr2.records])
print("launches", dp.info()["launches"], "resolve fallbacks", dp.info()["resolve_fallbacks"])

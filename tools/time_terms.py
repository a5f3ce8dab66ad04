"""Time one power-series term (pv_bench_terms) on a BASELINE config; PV_LIB_PATH picks a build,
PV_KNOBS="k=v,..." sets pv_set_option knobs first.
Usage: [PV_LIB_PATH=...] [PV_KNOBS=8=2] python tools/time_terms.py [config] [stage]"""
import os
import sys

sys.path.insert(0, os.getcwd())
import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
for kv in filter(None, os.environ.get("PV_KNOBS", "").split(",")):
    k, v = kv.split("=")
    dp.set_option(int(k), int(v))
st = synth.random_state(problem, 1)
if stage == 2:
    st, _ = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=3), dp=dp)
    st = pv.lift_stage1_to_stage2(st)
dp.set_state(st)
dp.linearize(stage)
dp.damp(1e-4, stage == 2)
dp.bench_terms(stage, 3)
tag = f"{os.path.basename(os.environ.get('PV_LIB_PATH', 'default'))} {os.environ.get('PV_KNOBS', '')}"
for _ in range(2):
    r = dp.bench_terms(stage, 10)
    print(tag, {k: round(v, 4) for k, v in r.items()}, flush=True)

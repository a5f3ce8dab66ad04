"""Sweep the term-kernel tuning knobs on a BASELINE config (results are knob-independent).
Usage: BLOCKS=32,48,64 POLS=122,000 DISC=1 python tools/sweep_terms.py [config] [stage]"""
import itertools
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
problem, _ = synth.make_problem(cfg_name, 0)
state = synth.random_state(problem, 1)
dp = pv.DeviceProblem(problem, 0.1)
if stage == 2:
    final, _ = pv.lm_minimize(problem, state, 1, pv.SolverConfig(max_outer_iterations=3), dp=dp)
    state = pv.lift_stage1_to_stage2(final)
dp.set_state(state)
dp.linearize(stage)
dp.damp(1e-4, stage == 2)
dp.power_solve(1, 0.0)
n_o = problem.num_observations
blocks = [int(c) for c in os.environ.get("BLOCKS", "32,48,64,96,4096").split(",")]
pols = [tuple(int(x) for x in p) for p in os.environ.get("POLS", "122,000").split(",")]
discs = [int(x) for x in os.environ.get("DISC", "1,0").split(",")]
for mb, (ps, pt, pss), disc in itertools.product(blocks, pols, discs):
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, mb << 20)
    dp.linearize(stage)  # re-blocking reorders the camera-sorted arrays
    dp.damp(1e-4, stage == 2)
    dp.power_solve(1, 0.0)
    dp.set_option(_lib.PV_OPT_POL_STREAM, ps)
    dp.set_option(_lib.PV_OPT_POL_T, pt)
    dp.set_option(_lib.PV_OPT_POL_S, pss)
    dp.set_option(_lib.PV_OPT_DISCARD_S, disc)
    dp.bench_terms(stage, 2)
    r = dp.bench_terms(stage, 10)
    print(f"block={mb:5d}MB B={dp.info()['blocks']:3d} pol={ps}{pt}{pss} disc={disc}  "
          f"lm_reduce~{r['lm_reduce_ms']:.3f} cam~{r['cam_ms']:.3f} term={r['term_ms']:.3f} ms  "
          f"{n_o / r['term_ms'] / 1e6:.2f} Gobs/s", flush=True)

"""A/B the term kernels under pv_set_option settings, interleaved on one context.
Usage: AB="7=0|7=1" ROUNDS=3 python tools/ab_terms.py [config] [stage]
Each variant is a comma list of key=value pv_set_option pairs; the power solve of
every variant is checked against the first one (results must be knob-independent)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
stage = int(sys.argv[2]) if len(sys.argv) > 2 else 1
variants = [[tuple(int(x) for x in kv.split("=")) for kv in v.split(",") if kv]
            for v in os.environ.get("AB", "7=0|7=1").split("|")]
rounds = int(os.environ.get("ROUNDS", "3"))
problem, _ = synth.make_problem(name, 0)
state = synth.random_state(problem, 1)
dp = pv.DeviceProblem(problem, 0.1)
if stage == 2:
    final, _ = pv.lm_minimize(problem, state, 1, pv.SolverConfig(max_outer_iterations=3), dp=dp)
    state = pv.lift_stage1_to_stage2(final)
dp.set_state(state)
dp.linearize(stage)
dp.damp(1e-4, stage == 2)
ref = None
res = {i: [] for i in range(len(variants))}
for rnd in range(rounds):
    for i, var in enumerate(variants):
        for k, v in var:
            dp.set_option(k, v)
        dp.linearize(stage)  # some knobs rebuild the work lists
        dp.damp(1e-4, stage == 2)
        order, trunc = dp.power_solve(30, 0.01)
        dx = dp.step(stage)[0].copy()
        if ref is None:
            ref = (order, dx)
        else:
            err = np.linalg.norm(dx - ref[1]) / np.linalg.norm(ref[1])
            assert order == ref[0] and err < 1e-12, (i, order, ref[0], err)
        dp.bench_terms(stage, 2)
        r = dp.bench_terms(stage, 10)
        res[i].append(r["term_ms"])
        print(f"round {rnd} variant {i} {var}: term {r['term_ms']:.4f} ms "
              f"(lm_reduce~{r['lm_reduce_ms']:.3f} cam~{r['cam_ms']:.3f})", flush=True)
for i, var in enumerate(variants):
    print(f"variant {i} {var}: best term {min(res[i]):.4f} ms  mean {np.mean(res[i]):.4f}")

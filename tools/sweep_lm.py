"""LM-iteration time (bench.py's value loop: iterations 1..K from the random start) under
pv_set_option settings.  Usage: python tools/sweep_lm.py [config] [K] "k=v,k=v|k=v|..."
Each '|'-separated variant is applied to the same context; the iterations restart from the
same state, so orders / accept decisions must agree across variants (checked)."""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 8
variants = [[tuple(int(x) for x in kv.split("=")) for kv in v.split(",") if kv]
            for v in (sys.argv[3] if len(sys.argv) > 3 else "").split("|")]
cfg = synth.CONFIGS[name]
problem, _ = synth.make_problem(name, 0)
state0 = synth.random_state(problem, 1)
dp = pv.DeviceProblem(problem, 0.1)
stream = torch.cuda.ExternalStream(dp.stream_handle)
scfg = pv.SolverConfig(max_power_order=cfg.max_power_order)


def run(k):
    dp.set_state(state0)
    f, lam, lin, orders = dp.cost(1), scfg.initial_lambda, False, []
    tt = 0
    for _ in range(k):
        if not lin:
            dp.linearize(1)
            lin = True
        dp.damp(lam, False)
        o, _ = dp.power_solve(scfg.max_power_order, scfg.power_threshold)
        inf = dp.info()
        tt += inf["solve_terms_us"] / max(1, inf["solve_terms_launched"])
        orders.append(o)
        ft = dp.cost(1, trial=True) if dp.trial(1) else math.inf
        if ft < f:
            f, _ = dp.accept(1, resolve=True)
            lin = False
            lam = max(scfg.lambda_min, lam * scfg.lambda_decrease)
        else:
            lam = min(scfg.lambda_max, lam * scfg.lambda_increase)
    return orders, f, tt / k


ref = None
for rnd in range(2):
    for var in variants:
        for kk, v in var:
            dp.set_option(kk, v)
        run(3)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        orders, f, us_term = run(K)
        e1.record(stream)
        torch.cuda.synchronize()
        if ref is None:
            ref = (orders, f)
        same = orders == ref[0] and abs(f - ref[1]) <= 1e-9 * abs(ref[1])
        info = dp.info()
        print(f"round {rnd} {var}: {e0.elapsed_time(e1) / K:.3f} ms/iteration, "
              f"{us_term / 1e3:.4f} ms/term (B={info['blocks']}), orders {orders} "
              f"{'same' if same else 'DIFFERENT'}", flush=True)

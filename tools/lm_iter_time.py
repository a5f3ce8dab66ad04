"""Time stage-1 LM iterations exactly as bench.py's `value` loop does (3 warm-up + K timed,
CUDA events on the library stream), for A/B of builds: PV_LIB_PATH=... python
tools/lm_iter_time.py [config] [K] [PV_OPT_x=v ...]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = synth.CONFIGS[name]
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
from paper_2405_05079_b200 import _lib  # noqa: E402
for kv in sys.argv[3:]:  # e.g. PV_OPT_SERIES=0
    k, v = kv.split("=")
    dp.set_option(getattr(_lib, k), int(v))
stream = torch.cuda.ExternalStream(dp.stream_handle)
scfg = pv.SolverConfig(max_outer_iterations=1, max_power_order=cfg.max_power_order,
                       function_tolerance=1e-300)
dp.set_state(synth.random_state(problem, 1))
f = dp.cost(1)
lam = scfg.initial_lambda
orders, acc = [], []


lin = [False]


def it():
    # as solver.lm_minimize / bench.py: re-linearize only after an accepted step
    global f, lam
    if not lin[0]:
        dp.linearize(1)
        lin[0] = True
    dp.damp(lam, False)
    o, _ = dp.power_solve(scfg.max_power_order, scfg.power_threshold)
    orders.append(o)
    ok = dp.trial(1)
    ft = dp.cost(1, trial=True) if ok else math.inf
    if ft < f:
        f, _ = dp.accept(1, resolve=True)
        lin[0] = False
        lam = max(scfg.lambda_min, lam * scfg.lambda_decrease)
        acc.append(1)
    else:
        lam = min(scfg.lambda_max, lam * scfg.lambda_increase)
        acc.append(0)


for _ in range(3):
    it()
orders.clear()
acc.clear()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(stream)
for _ in range(K):
    it()
e1.record(stream)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / K
print(f"{os.environ.get('PV_LIB_PATH', 'default')} {' '.join(sys.argv[3:])}: {ms:.3f} ms/iteration, orders {orders}, "
      f"accepted {sum(acc)}/{K}, cost {f!r}")

"""Term time vs the work-list balance of the persistent camera kernel (PV_OPT_BALANCE and its
cost model, PV_OPT_BAL_ITEM / _ROUND / _LAST) on a BASELINE config; also checks that every
setting gives the same power-series bits.
Usage: [PV_DEBUG_BALANCE=1] python tools/sweep_balance.py [config] ["mode:item:round:last[:kslot],..."]"""
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
combos = sys.argv[2] if len(sys.argv) > 2 else "0:24:0:0,1:24:0:0,1:48:0:0,1:24:32:0,1:48:32:32,1:96:0:0,0:24:0:0,1:24:0:0"
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
dp.linearize(1)
dp.damp(1e-4, False)
for cb in combos.split(","):
    f = [int(x) for x in cb.split(":")]
    mode, item, rnd, last = f[:4]
    if len(f) > 4:  # optional fifth field: PV_OPT_KSLOT
        dp.set_option(_lib.PV_OPT_KSLOT, f[4])
    dp.set_option(_lib.PV_OPT_BAL_ITEM, item)
    dp.set_option(_lib.PV_OPT_BAL_ROUND, rnd)
    dp.set_option(_lib.PV_OPT_BAL_LAST, last)
    dp.set_option(_lib.PV_OPT_BALANCE, mode)
    dp.power_solve(6, 0.0)
    h = hashlib.sha256(dp.debug(_lib.PV_DBG_X).tobytes()).hexdigest()[:12]
    dp.bench_terms(1, 3)
    r = dp.bench_terms(1, 20)
    print(f"balance {cb}: lm_reduce~{r['lm_reduce_ms']:.4f} cam~{r['cam_ms']:.4f} "
          f"term {r['term_ms']:.4f} ms  dx {h}", flush=True)

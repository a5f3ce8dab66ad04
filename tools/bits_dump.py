"""Hash of the power-solve results (tiny with 64 KB blocks and the small config, stages 1 and
2) for bit-identity comparisons between builds: PV_LIB_PATH=... python tools/bits_dump.py"""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

h = hashlib.sha256()
for name, bb in (("tiny", 64 << 10), ("small", 256 << 10), ("medium", 8 << 20)):
    problem, _ = synth.make_problem(name, 0)
    st = synth.random_state(problem, 1)
    dp = pv.DeviceProblem(problem, 0.1)
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, bb)
    s1, tr = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=4), dp=dp)
    for r in tr.records:
        h.update(repr(r.cost).encode())
    h.update(s1.cameras.tobytes())
    h.update(s1.landmarks.tobytes())
    s2, tr2 = pv.lm_minimize(problem, pv.lift_stage1_to_stage2(s1), 2,
                             pv.SolverConfig(max_outer_iterations=2), dp=dp)
    h.update(s2.cameras.tobytes())
    h.update(s2.landmarks.tobytes())
print(os.path.basename(os.environ.get("PV_LIB_PATH", "default")), h.hexdigest())

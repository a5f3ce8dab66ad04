"""Host <-> device state transfer times of the public API on a BASELINE config
(pv_set_state / pv_get_state, what lm_minimize pays once per call)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
st = synth.random_state(problem, 1)
mb = (st.cameras.nbytes + st.landmarks.nbytes) / 1e6
for rep in range(3):
    t0 = time.perf_counter(); dp.set_state(st); t1 = time.perf_counter()
    out = dp.get_state(); t2 = time.perf_counter()
    f = dp.cost(1); t3 = time.perf_counter()
    print(f"{mb:.0f} MB: set_state {1e3 * (t1 - t0):.2f} ms, get_state {1e3 * (t2 - t1):.2f} ms, cost {1e3 * (t3 - t2):.2f} ms", flush=True)
assert np.array_equal(out.landmarks, st.landmarks) and np.array_equal(out.cameras, st.cameras)

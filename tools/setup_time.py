import sys, time, os
sys.path.insert(0, os.getcwd())
import paper_2405_05079_b200 as pv
from paper_2405_05079_b200 import synth
problem, _ = synth.make_problem("vlarge", 0)
for i in range(2):
    t = time.perf_counter(); dp = pv.DeviceProblem(problem, 0.1); print("DeviceProblem", time.perf_counter() - t, flush=True); del dp

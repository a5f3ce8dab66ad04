"""A small end-to-end driver for compute-sanitizer (tools/sanitize.sh): every kernel family
of libpovar.so on the tiny config with 64 KB landmark blocks (several blocks, one warp per
camera -> the TMA-pipelined camera kernel, the compact stage-1 stream and the CUDA-graph
term loop), stage 1 and 2, power and PCG, the landmark re-solve, back-substitution, the
host-loop variant and a 2-rank loopback run.
Usage: python tools/sanitize_case.py [--no-loopback]"""
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, shard, synth  # noqa: E402

problem, _ = synth.make_problem("tiny", 0)
st = synth.random_state(problem, 1)
for graph in (1, 0):
    dp = pv.DeviceProblem(problem, 0.1)
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, 64 << 10)
    dp.set_option(_lib.PV_OPT_GRAPH, graph)
    info = dp.info()
    assert info["blocks"] > 1 and info["warps_per_cam"] == 1, info
    s1, tr1 = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=3), dp=dp)
    s2, tr2 = pv.lm_minimize(problem, pv.lift_stage1_to_stage2(s1), 2,
                             pv.SolverConfig(max_outer_iterations=2), dp=dp)
    _, trp = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=2,
                                                           inner_solver="pcg"), dp=dp)
    sysm = pv.assemble_system(problem, s1, 1, 1e-3, "pose_only", dp=dp)
    pv.back_substitute(sysm, np.ones(sysm.pose_dim))
    print(f"graph={graph}: stage-1 costs {[r.cost for r in tr1.records]}, "
          f"stage-2 {[r.cost for r in tr2.records]}, pcg {[r.cost for r in trp.records]}")
    dp.close()
if "--no-loopback" not in sys.argv:
    world = 2
    plan = shard.plan_shards(problem, world)
    lid = shard.loopback_id(world)
    dps = [pv.DeviceProblem(problem, 0.1, rank=r, world=world, nccl_id=lid, lm_range=plan[r])
           for r in range(world)]
    out = [None] * world

    def run(r):
        out[r] = pv.lm_minimize(problem, st, 1, pv.SolverConfig(max_outer_iterations=2),
                                dp=dps[r])

    th = [threading.Thread(target=run, args=(r,), daemon=True) for r in range(world)]
    [t.start() for t in th]
    [t.join(timeout=600) for t in th]
    assert all(o is not None for o in out)
    print("loopback costs", [r.cost for r in out[0][1].records])
    for d in dps:
        d.close()
print("SANITIZE_CASE_OK")

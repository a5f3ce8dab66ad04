"""Term time vs the landmark-block L2 budget (PV_OPT_BLOCK_BYTES) on a BASELINE config.
Usage: [PV_LIB_PATH=...] python tools/sweep_blocks.py [config] [MB,MB,...]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2405_05079_b200 as pv  # noqa: E402
from paper_2405_05079_b200 import _lib, synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "vlarge"
mbs = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "48,64,80").split(",")]
problem, _ = synth.make_problem(name, 0)
dp = pv.DeviceProblem(problem, 0.1)
dp.set_state(synth.random_state(problem, 1))
for mb in mbs:
    dp.set_option(_lib.PV_OPT_BLOCK_BYTES, mb << 20)
    dp.linearize(1)
    dp.damp(1e-4, False)
    dp.bench_terms(1, 3)
    r = dp.bench_terms(1, 10)
    info = dp.info()
    print(f"{os.environ.get('PV_LIB_PATH', 'default')} budget {mb} MB: B={info['blocks']} "
          f"wpc={info['warps_per_cam']} lm_reduce~{r['lm_reduce_ms']:.4f} cam~{r['cam_ms']:.4f} "
          f"term {r['term_ms']:.4f} ms", flush=True)

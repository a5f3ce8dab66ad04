#!/bin/bash
# A/B of the camera-pass kernels + the variant tests (run under gpurun from the repo root)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -q -x > gpurun_out/variants.log 2>&1
echo "variants rc=$?" >> gpurun_out/variants.log
AB="${AB:-8=1|8=2}" ROUNDS=3 timeout 900 python tools/ab_terms.py vlarge 1 > gpurun_out/ab1.log 2>&1
AB="${AB:-8=1|8=2}" ROUNDS=2 timeout 900 python tools/ab_terms.py vlarge 2 > gpurun_out/ab2.log 2>&1
tail -3 gpurun_out/variants.log; tail -3 gpurun_out/ab1.log; tail -3 gpurun_out/ab2.log

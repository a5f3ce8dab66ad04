#!/bin/bash
# One GPU-box pass: all -m gpu tests (no -x: every failure reported, achieved parity
# errors to gpurun_out/parity.json), smoke, then the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
PV_PARITY_REPORT=gpurun_out/parity.json timeout 1500 python -m pytest tests -m gpu -q -s -rf \
  > gpurun_out/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
if [ "${BENCH:-1}" = 1 ]; then
  timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench rc=$?" >> gpurun_out/bench.err
fi
tail -5 gpurun_out/pytest.log; tail -2 gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench.json

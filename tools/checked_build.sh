#!/bin/bash
# Checked builds of libpovar.so (compute-sanitizer is not available on the GPU pool):
#   build_ab/libpovar_checked.so  -DPV_CHECKED: device bounds / invariant checks (PV_CHECK)
#   build_ab/libpovar_fence.so    -DPV_PIPE_FENCE=1: proxy fence before every TMA refill
# Run on the GPU box: bash tools/checked_build.sh run
cd "$(dirname "$0")/.."
if [ "$1" = run ]; then
  mkdir -p gpurun_out
  PV_LIB_PATH=$PWD/build_ab/libpovar_checked.so timeout 1500 python -m pytest tests -m gpu -q \
    -x > gpurun_out/checked_pytest.log 2>&1; echo "checked pytest rc=$?" >> gpurun_out/checked_pytest.log
  PV_LIB_PATH=$PWD/build_ab/libpovar_checked.so timeout 600 python tools/sanitize_case.py \
    > gpurun_out/checked_case.log 2>&1; echo "checked case rc=$?" >> gpurun_out/checked_case.log
  PV_LIB_PATH=$PWD/build_ab/libpovar_fence.so timeout 900 python -m pytest \
    tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/fence_pytest.log 2>&1
  echo "fence pytest rc=$?" >> gpurun_out/fence_pytest.log
  for lib in default fence checked; do
    if [ $lib = default ]; then unset PV_LIB_PATH; else export PV_LIB_PATH=$PWD/build_ab/libpovar_$lib.so; fi
    timeout 600 python tools/bits_dump.py >> gpurun_out/bits.log 2>&1
  done
  unset PV_LIB_PATH
  for lib in default fence; do
    if [ $lib = default ]; then unset PV_LIB_PATH; else export PV_LIB_PATH=$PWD/build_ab/libpovar_$lib.so; fi
    timeout 600 python tools/time_terms.py vlarge >> gpurun_out/fence_time.log 2>&1
  done
  tail -3 gpurun_out/checked_pytest.log gpurun_out/checked_case.log gpurun_out/fence_pytest.log
  cat gpurun_out/bits.log; grep -v Warn gpurun_out/fence_time.log
  exit 0
fi
tools/build_variants.sh "checked:-DPV_CHECKED" "fence:-DPV_PIPE_FENCE=1"

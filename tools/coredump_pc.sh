#!/bin/bash
# Run a command with GPU core dumps enabled and print where the device exception hit
# (kernel, PC, SASS around it).  Usage (under gpurun): tools/coredump_pc.sh <command...>
rm -f gpurun_out/gpucore*
export CUDA_ENABLE_COREDUMP_ON_EXCEPTION=1
export CUDA_COREDUMP_FILE=gpurun_out/gpucore
export CUDA_COREDUMP_GENERATION_FLAGS="skip_global_memory,skip_shared_memory,skip_local_memory,skip_constbank_memory"
"$@" > gpurun_out/coredump_cmd.log 2>&1
echo "command rc=$?"; ls -la gpurun_out/gpucore* 2>/dev/null
f=$(ls gpurun_out/gpucore* 2>/dev/null | head -1)
[ -n "$f" ] && timeout 300 cuda-gdb -batch -ex "target cudacore $f" -ex "info cuda kernels" \
  -ex "info cuda lanes" -ex "x/12i \$errorpc-64" -ex "x/6i \$errorpc" -ex "info registers \$errorpc" 2>&1 | tail -60
rm -f gpurun_out/gpucore*

#!/bin/bash
# Round measurement (run under gpurun from the repo root): bench (both arms), launch list,
# warm per-term DRAM traffic, and a full ncu capture of the term kernels; outputs in gpurun_out/.
# profile_terms.py launches (vlarge, B = 12): 1 seed W^T v pass, then per term 12 landmark
# reduces + 11 k_cam_pipe<1,1,1> + 1 k_cam_pipe<1,1,0> (last block's W t) + 1 k_cam
# (epilogue) + 1 k_cam_pipe<1,0,1> (next term's W^T v of block 0) = 26 launches.
# NCU_ONLY=1 skips the bench runs.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
if [ -z "$NCU_ONLY" ]; then
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
fi
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
    --no-e2e > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
python tools/profile_terms.py vlarge 1 4 > gpurun_out/plain2.log 2>&1 && \
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --cache-control none --clock-control none -k regex:"k_cam|k_lm_reduce" -s 27 -c 26 --csv \
    --log-file gpurun_out/traffic.csv python tools/profile_terms.py vlarge 1 4 \
    > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"k_cam_pipe|k_lm_reduce" -s 26 -c 2 -o gpurun_out/prof_term \
  python tools/profile_terms.py vlarge 1 3 > gpurun_out/ncu3.log 2>&1; echo ncu3=$?

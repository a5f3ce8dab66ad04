#!/bin/bash
# ncu --set full capture of one steady-state camera-pass launch (vlarge, stage 1), source-level.
# Usage (under gpurun): bash tools/ncu_pipe.sh <tag> [knobs, e.g. 8=2]
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${1:-pipe}; KN=${2:-}
python tools/profile_terms.py vlarge 1 2 $KN > gpurun_out/plain_$TAG.log 2>&1 || exit 1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on \
  -k regex:"k_cam_pipe" -s 30 -c 1 -o gpurun_out/prof_$TAG \
  python tools/profile_terms.py vlarge 1 3 $KN > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?

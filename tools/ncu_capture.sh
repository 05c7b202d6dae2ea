#!/bin/bash
# one --set full capture per kernel name of one hot-path step: tools/ncu_capture.sh TAG K1 [K2 ...]
set -e
TAG=$1; shift
mkdir -p gpurun_out
python tools/profile_step.py --steps 1 > gpurun_out/cap_step_$TAG.log
for K in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o gpurun_out/cap_${K}_$TAG -f python tools/profile_step.py --steps 1 > gpurun_out/cap_${K}_$TAG.log 2>&1
done

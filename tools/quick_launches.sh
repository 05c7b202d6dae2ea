#!/bin/bash
# launch list (cold, serialised) of 2 hot-path steps of a config; summary to stdout
set -e
TAG=${1:-q}
shift || true
mkdir -p gpurun_out
python tools/profile_step.py --steps 2 "$@" > gpurun_out/qstep_$TAG.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qlaunch_$TAG.csv \
    python tools/profile_step.py --steps 2 "$@" > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/qlaunch_$TAG.csv > gpurun_out/qsum_$TAG.md
head -45 gpurun_out/qsum_$TAG.md

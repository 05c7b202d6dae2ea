#!/bin/bash
# ncu evidence for one round (run on the GPU box from the repo root):
#  1. launch list of the bench command (per-launch durations, cold, serialised)
#  2. one --set full capture of the dominant kernels of one hot-path step
# Each profiled command is first run once without ncu and must exit 0.
set -e
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_small_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_bench_$TAG.log 2>&1
python tools/profile_step.py --steps 1 > $OUT/step_$TAG.log
for K in ${KERNELS:-schur_trailing_kernel}; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c ${COUNT:-1} \
      -o $OUT/full_${K}_$TAG -f python tools/profile_step.py --steps 1 > $OUT/ncu_full_${K}_$TAG.log 2>&1
done

#!/bin/bash
# ncu evidence (run on the GPU box from the repo root): launch list of the
# bench command + --set full captures of the dominant setup kernel (all six
# trailing launches of one elimination) and of the apply kernels.
set -e
TAG=${1:-r01b}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_small_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_bench_$TAG.log 2>&1
python tools/profile_step.py --steps 1 > $OUT/step_$TAG.log
ncu --set full --clock-control none --import-source on -k regex:schur_trailing_kernel -c 6 \
    -o $OUT/full_trailing_$TAG -f python tools/profile_step.py --steps 1 > $OUT/ncu_full_trailing_$TAG.log 2>&1
for K in local_solve_kernel local_gemv_kernel coarse_blk_solve_kernel face_fast_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o $OUT/full_${K}_$TAG -f python tools/profile_step.py --steps 1 > $OUT/ncu_full_${K}_$TAG.log 2>&1
done

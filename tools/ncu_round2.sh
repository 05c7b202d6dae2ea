#!/bin/bash
# ncu evidence (run on the GPU box from the repo root): launch list of the
# bench command + --set full captures of the dominant setup kernel (the
# trailing launches of one step) and of the apply kernels.  The reports are
# summarised on the box (ncu_summary.py, traffic.py) and only the small ones
# are kept, so gpurun_out/ stays below the copy-back limit.
set -e
TAG=${1:-r01b}
OUT=gpurun_out
mkdir -p $OUT
python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/bench_small_$TAG.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 1 --warmup 3 --e2e-steps 1 --no-cpu-baseline > $OUT/ncu_bench_$TAG.log 2>&1
python tools/profile_step.py --steps 1 > $OUT/step_$TAG.log
ncu --set full --clock-control none --import-source on -k regex:schur_trailing_kernel -c 16 \
    -o $OUT/full_trailing_$TAG -f python tools/profile_step.py --steps 1 > $OUT/ncu_full_trailing_$TAG.log 2>&1
python tools/traffic.py $OUT/full_trailing_$TAG.ncu-rep $TAG > $OUT/traffic_$TAG.log 2>&1 || true
REPS=$OUT/full_trailing_$TAG.ncu-rep
for K in local_solve_kernel local_gemv_kernel coarse_blk_solve_kernel face_fast_kernel gj_update_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:$K -c 1 \
      -o $OUT/full_${K}_$TAG -f python tools/profile_step.py --steps 1 > $OUT/ncu_full_${K}_$TAG.log 2>&1
  REPS="$REPS $OUT/full_${K}_$TAG.ncu-rep"
done
python tools/ncu_summary.py $OUT/launches_$TAG.csv $REPS > $OUT/ncu_summary_$TAG.md 2>&1 || true
cp profiles/trailing_traffic_$TAG.json $OUT/ 2>/dev/null || true
rm -f $OUT/full_trailing_$TAG.ncu-rep $OUT/full_face_fast_kernel_$TAG.ncu-rep $OUT/full_gj_update_kernel_$TAG.ncu-rep

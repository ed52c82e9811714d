#!/bin/bash
# C5 batched: value sets per lane per iteration of the batched specialised kernels (SGB_BATCH_VEC).
TAG=${1:-bvec}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for V in 4 2 8 4 8; do
  SGB_BATCH_VEC=$V timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline \
     >> $OUT/bench_c5_v$V.json 2>> $OUT/bench_c5_v$V.err
  echo "c5 vec $V rc=$?" >> $OUT/status.txt
done

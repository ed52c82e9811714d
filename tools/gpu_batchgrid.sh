#!/bin/bash
# C5 batched: persistent vs one-block-per-tile grid for the batched specialised kernels.
TAG=${1:-bgrid}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for G in persistent tiles persistent tiles; do
  SGB_BATCH_GRID=$G timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline \
     >> $OUT/bench_c5_$G.json 2>> $OUT/bench_c5_$G.err
  echo "c5 $G rc=$?" >> $OUT/status.txt
done

#!/bin/bash
TAG=${1:-r2z}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( timeout 900 python bench.py --config c1 --only --no-cpu-baseline ) > $OUT/c1.json 2> $OUT/c1.err; echo "c1 rc=$?" >> $OUT/status.txt
for W in 2 4 8; do
  timeout 900 python bench.py --split outputs --split-world $W --split-rank 0 --steps 20 --warmup 3 --no-cpu-baseline \
     > $OUT/bench_c2_split${W}_r0.json 2> $OUT/bench_c2_split${W}_r0.err
  echo "split $W rc=$?" >> $OUT/status.txt
done

#!/bin/bash
TAG=${1:-c5fix}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 1500 python -m pytest tests -m gpu -x -q -k "batch or host_many or shards" ) > $OUT/pytest_batch.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for V in 4 4 8; do
  SGB_BATCH_VEC=$V timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline \
     >> $OUT/bench_c5_v$V.json 2>> $OUT/bench_c5_v$V.err
  echo "c5 vec $V rc=$?" >> $OUT/status.txt
done

#!/bin/bash
# Output sharding: GPU parity of the shard plans, and one rank's share of a 2/4/8-way C2 output split
# timed on one B200 (the N-GPU job runs each share on its own GPU, no collective in the step).
TAG=${1:-split}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 1500 python -m pytest tests -m gpu -x -q -k "output_shards or host_many or tile_schedules" ) > $OUT/pytest_split.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for W in 2 4 8; do
  for R in 0 $((W-1)); do
    timeout 900 python bench.py --split outputs --split-world $W --split-rank $R --steps 20 --warmup 3 \
       > $OUT/bench_c2_split${W}_r$R.json 2> $OUT/bench_c2_split${W}_r$R.err
    echo "split $W rank $R rc=$?" >> $OUT/status.txt
  done
done

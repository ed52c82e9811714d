#!/bin/bash
# Output gather variants: capped grid-stride (default), one block per 256 outputs, four outputs per thread.
TAG=${1:-gather}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for C in c2 c3; do
  for V in default tiles v4 default v4; do
    case $V in tiles) E="SGB_GATHER_GRID=tiles";; v4) E="SGB_GATHER=v4";; *) E="SGB_NONE=1";; esac
    env $E timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline \
       >> $OUT/bench_${C}_$V.json 2>> $OUT/bench_${C}_$V.err
    echo "$C $V rc=$?" >> $OUT/status.txt
  done
done

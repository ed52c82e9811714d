#!/bin/bash
TAG=${1:-r3c}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( timeout 900 python bench.py --config c1 --only --no-cpu-baseline ) > $OUT/c1.json 2> $OUT/c1.err; echo "c1 rc=$?" >> $OUT/status.txt
( timeout 900 python bench.py --only --no-cpu-baseline ) > $OUT/c2.json 2> $OUT/c2.err; echo "c2 rc=$?" >> $OUT/status.txt

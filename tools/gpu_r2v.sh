#!/bin/bash
TAG=${1:-r2v}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/c5_variants.py > $OUT/c5.log 2>&1; echo "c5 rc=$?" >> $OUT/status.txt
( timeout 900 python bench.py --only --steps 20 --no-cpu-baseline ) > $OUT/c2.json 2> $OUT/c2.err; echo "c2 rc=$?" >> $OUT/status.txt

#!/bin/bash
TAG=${1:-r2q}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/c5_variants.py > $OUT/c5.log 2>&1; echo "c5 rc=$?" >> $OUT/status.txt
timeout 900 python tools/vec_variants.py > $OUT/vec.log 2>&1; echo "vec rc=$?" >> $OUT/status.txt

#!/bin/bash
TAG=${1:-r3k}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/win_variants.py > $OUT/win_variants.log 2>&1; echo "win rc=$?" >> $OUT/status.txt
timeout 900 python tools/c5_bvec.py > $OUT/c5_bvec.log 2>&1; echo "c5 rc=$?" >> $OUT/status.txt

#!/bin/bash
TAG=${1:-r3f}; OUT=gpurun_out/$TAG; mkdir -p $OUT
bash tools/gpu_check.sh $TAG
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/win_variants.py > $OUT/win_variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt

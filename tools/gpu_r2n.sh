#!/bin/bash
TAG=${1:-r2n}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 1500 python tools/index_variants.py > $OUT/index.log 2>&1; echo "index rc=$?" >> $OUT/status.txt

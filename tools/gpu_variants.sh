#!/bin/bash
# Run one variant harness on the GPU box:  bash tools/gpu_variants.sh TAG tools/win_variants.py [args]
TAG=${1:-var}; SCRIPT=$2; shift 2; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 1500 python $SCRIPT "$@" > $OUT/$(basename $SCRIPT .py).log 2>&1; echo "$SCRIPT rc=$?" >> $OUT/status.txt

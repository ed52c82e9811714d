#!/bin/bash
# C3 element-kernel variants.   bash tools/gpu_c3v.sh TAG
TAG=${1:-c3v}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python tools/c3_variants.py > $OUT/c3_variants.log 2>&1; echo "c3 rc=$?" >> $OUT/status.txt

#!/bin/bash
# C3 element-kernel variants + C2 window load depth.   bash tools/gpu_r2h.sh TAG
TAG=${1:-r2h}; OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python tools/c3_variants.py > $OUT/c3_variants.log 2>&1; echo "c3 rc=$?" >> $OUT/status.txt
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt

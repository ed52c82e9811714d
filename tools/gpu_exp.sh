#!/bin/bash
# Experiment: variants + ncu full capture of one launch.  bash tools/gpu_exp.sh TAG VARIANTS NCU_FILTER SKIP
TAG=${1:-e}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/variants.py 1000 "$2" > $OUT/variants.log 2>&1
echo "variants rc=$?" >> $OUT/status.txt
if [ -n "$3" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$3" -s ${4:-4} -c 1 \
   -o $OUT/prof python tools/profile_run.py --evals 3 > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/status.txt
fi

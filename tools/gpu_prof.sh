#!/bin/bash
# ncu --set full over the kernels of evaluations 2..N (launch list + full metrics).  bash tools/gpu_prof.sh TAG MODE SKIP COUNT
TAG=${1:-p}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 600 python tools/profile_run.py --evals 1 --mode ${2:-csr} > $OUT/units.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"sop|tape|gather" -s ${3:-12} -c ${4:-12} \
   -o $OUT/prof python tools/profile_run.py --evals 3 --mode ${2:-csr} > $OUT/ncu.log 2>&1
echo "ncu rc=$?" >> $OUT/status.txt

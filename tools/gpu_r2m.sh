#!/bin/bash
TAG=${1:-r2m}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgb_wbulk -s 1 -c 1 \
   -o $OUT/wbulk python tools/profile_run.py --config c2 --evals 3 --wbulk on > $OUT/ncu_wbulk.log 2>&1
echo "ncu rc=$?" >> $OUT/status.txt
( timeout 900 python bench.py --config c3 --only --steps 10 --no-cpu-baseline ) > $OUT/c3.json 2> $OUT/c3.err
echo "c3 rc=$?" >> $OUT/status.txt

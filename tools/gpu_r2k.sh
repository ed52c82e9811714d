#!/bin/bash
# Bulk window: ncu of the bulk kernel, variants; C3 round-1 code vs now.
TAG=${1:-r2k}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgb_wbulk -s 1 -c 1 \
   -o $OUT/wbulk python tools/profile_run.py --config c2 --evals 3 --wbulk on > $OUT/ncu_wbulk.log 2>&1
echo "ncu rc=$?" >> $OUT/status.txt
( cd _scratch_r1 && timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline ) > $OUT/c3_r1code.json 2> $OUT/c3_r1code.err
echo "c3 r1 rc=$?" >> $OUT/status.txt

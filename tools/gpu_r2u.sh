#!/bin/bash
TAG=${1:-r2u}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 python tools/c5_variants.py > $OUT/c5.log 2>&1; echo "c5 rc=$?" >> $OUT/status.txt
for D in 0 1; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" --csv --log-file $OUT/launches_c5_direct$D.csv python tools/prof_c5.py $D > $OUT/ncu_c5_$D.log 2>&1
echo "ncu $D rc=$?" >> $OUT/status.txt
done

#!/bin/bash
# C5 batched: launch list and one ncu --set full capture of the batched specialised kernels.
TAG=${1:-c5prof}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 40 --csv --log-file $OUT/launches_c5.csv \
   python tools/profile_run.py --config c2 --w 200 --batch 256 --evals 2 > $OUT/ncu_launches_c5.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none -k regex:"sgb_tape_b|gather" -s 4 -c 3 \
   -o $OUT/prof_c5 python tools/profile_run.py --config c2 --w 200 --batch 256 --evals 2 > $OUT/ncu_full_c5.log 2>&1
echo "full rc=$?" >> $OUT/status.txt

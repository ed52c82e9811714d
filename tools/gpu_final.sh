#!/bin/bash
# Evidence pass: per config, the ncu launch list of a short evaluation loop and one --set full
# capture of its dominant kernel(s).  bash tools/gpu_final.sh TAG
TAG=${1:-final}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for C in c2 c3 c4; do
  timeout 900 python tools/profile_run.py --config $C --evals 1 > $OUT/units_$C.log 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"sgb|sop|tape|gather" -c 60 --csv --log-file $OUT/launches_$C.csv \
     python tools/profile_run.py --config $C --evals 3 > $OUT/ncu_launches_$C.log 2>&1
  echo "$C launches rc=$?" >> $OUT/status.txt
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape_u3|gather" -s 2 -c 2 \
   -o $OUT/prof_c2 python tools/profile_run.py --config c2 --evals 3 > $OUT/ncu_full_c2.log 2>&1
echo "c2 full rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape" -s 2 -c 2 \
   -o $OUT/prof_c3 python tools/profile_run.py --config c3 --evals 2 > $OUT/ncu_full_c3.log 2>&1
echo "c3 full rc=$?" >> $OUT/status.txt

#!/bin/bash
# CSR-layout check: GPU parity of the relaid plans, C3/C2/C4 bench in both layouts, ncu of C3's units.
TAG=${1:-lay}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 900 python -m pytest tests -m gpu -x -q -k "csr_layout" ) > $OUT/pytest_layout.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for C in c3 c2 c4; do
  for LAY in csr reference; do
    timeout 900 python bench.py --config $C --steps 10 --warmup 3 --layout $LAY --no-cpu-baseline > $OUT/bench_${C}_$LAY.json 2> $OUT/bench_${C}_$LAY.err
    echo "bench $C $LAY rc=$?" >> $OUT/status.txt
  done
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 40 --csv --log-file $OUT/launches_c3.csv \
   python tools/profile_run.py --config c3 --evals 3 > $OUT/ncu_launches_c3.log 2>&1
echo "ncu c3 rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape" -s 2 -c 2 \
   -o $OUT/prof_c3 python tools/profile_run.py --config c3 --evals 2 > $OUT/ncu_full_c3.log 2>&1
echo "c3 full rc=$?" >> $OUT/status.txt

#!/bin/bash
# Tile-order experiment: instance vs fraction interleave of specialised-unit tiles on C2/C3/C4,
# plus the C3 launch list (DRAM bytes per launch) under the fraction order.  bash tools/gpu_order.sh TAG
TAG=${1:-order}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for C in c2 c4 c3; do
  for O in inst frac; do
    SGB_TILE_ORDER=$O timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline \
       > $OUT/bench_${C}_$O.json 2> $OUT/bench_${C}_$O.err
    echo "bench $C $O rc=$?" >> $OUT/status.txt
  done
done
SGB_TILE_ORDER=frac timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 12 --csv --log-file $OUT/launches_c3_frac.csv \
   python tools/profile_run.py --config c3 --evals 3 > $OUT/ncu_launches_c3.log 2>&1
echo "ncu c3 rc=$?" >> $OUT/status.txt

#!/bin/bash
# Grid experiment: persistent grid-stride specialised units vs one block per tile (SGB_JIT_GRID=tiles)
# on C2/C3/C4, plus C3 launch lists (DRAM bytes) for both.   bash tools/gpu_grid.sh TAG
TAG=${1:-grid}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for C in c3 c2 c4; do
  for G in persistent tiles; do
    SGB_JIT_GRID=$G timeout 900 python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline \
       > $OUT/bench_${C}_$G.json 2> $OUT/bench_${C}_$G.err
    echo "bench $C $G rc=$?" >> $OUT/status.txt
  done
done
for G in persistent tiles; do
  SGB_JIT_GRID=$G timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     -k regex:"sgb|sop|tape|gather" -c 12 --csv --log-file $OUT/launches_c3_$G.csv \
     python tools/profile_run.py --config c3 --evals 3 --schedule frac > $OUT/ncu_launches_c3_$G.log 2>&1
  echo "ncu c3 $G rc=$?" >> $OUT/status.txt
done

#!/bin/bash
TAG=${1:-lay2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 900 python -m pytest tests -m gpu -x -q -k "csr_layout or specialised or graph" ) > $OUT/pytest_layout.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_csr.json 2> $OUT/bench_c3_csr.err
echo "bench c3 csr rc=$?" >> $OUT/status.txt
SGB_TILE_ORDER=frac timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $OUT/bench_c3_frac.json 2> $OUT/bench_c3_frac.err
echo "bench c3 frac rc=$?" >> $OUT/status.txt
SGB_TILE_ORDER=frac timeout 900 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --layout reference > $OUT/bench_c3_frac_ref.json 2> $OUT/bench_c3_frac_ref.err
echo "bench c3 frac ref rc=$?" >> $OUT/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 12 --csv --log-file $OUT/launches_c3.csv \
   python tools/profile_run.py --config c3 --evals 3 > $OUT/ncu_launches_c3.log 2>&1
echo "ncu c3 rc=$?" >> $OUT/status.txt

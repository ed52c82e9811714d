#!/bin/bash
# Round-end evidence: smoke, GPU parity suite, every config's bench line, the reference arm, the ncu
# launch list of the default bench command, and ncu --set full captures of the dominant kernels.
#   bash tools/gpu_evidence.sh TAG
TAG=${1:-ev}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo "bench c2 rc=$?" >> $OUT/status.txt
for C in ${CONFIGS:-c1 c3 c4 c5}; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "bench $C rc=$?" >> $OUT/status.txt
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference_c2.json 2> $OUT/bench_reference_c2.err
echo "reference rc=$?" >> $OUT/status.txt
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 400 --csv --log-file $OUT/launches_bench_c2.csv \
   python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench_c2.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape_u3|gather" -s 2 -c 2 \
   -o $OUT/prof_c2 python tools/profile_run.py --config c2 --evals 3 > $OUT/ncu_full_c2.log 2>&1
echo "full c2 rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape" -s 2 -c 2 \
   -o $OUT/prof_c3 python tools/profile_run.py --config c3 --evals 2 --schedule frac --grid tiles > $OUT/ncu_full_c3.log 2>&1
echo "full c3 rc=$?" >> $OUT/status.txt

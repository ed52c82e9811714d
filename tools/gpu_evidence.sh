#!/bin/bash
# Round evidence on one B200: smoke, the GPU suite, the default bench line (C2 + other_configs), the
# reference arm, the ncu launch list of the C2 bench command and ncu --set full captures of the
# dominant kernels (C2 window + wave0, C3 element kernel).     bash tools/gpu_evidence.sh TAG
TAG=${1:-ev}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
( time timeout 1500 python bench.py ) > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
echo "reference rc=$?" >> $OUT/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
   -k regex:"sgb|sop|tape|gather" -c 300 --csv --log-file $OUT/launches_bench_c2.csv \
   python bench.py --only --steps 3 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench_c2.log 2>&1
echo "launches rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_window|sgb_tape_u0" -s 2 -c 2 \
   -o $OUT/prof_c2 python tools/profile_run.py --config c2 --evals 3 > $OUT/ncu_full_c2.log 2>&1
echo "full c2 rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"sgb_tape_u0" -s 1 -c 1 \
   -o $OUT/prof_c3 python tools/profile_run.py --config c3 --evals 2 > $OUT/ncu_full_c3.log 2>&1
echo "full c3 rc=$?" >> $OUT/status.txt

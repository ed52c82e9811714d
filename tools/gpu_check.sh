#!/bin/bash
# One GPU session: smoke, GPU parity tests, bench, ncu launch list + one full capture.
# Usage (from the repo root, under gpurun): bash tools/gpu_check.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time python -c "import __graft_entry__ as g; g.build(); g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
   --log-file $OUT/launches.csv python tools/profile_run.py --evals 3 > $OUT/ncu_launches.log 2>&1
echo "ncu launches rc=$?" >> $OUT/status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sop|tape" -s 15 -c 15 \
   -o $OUT/prof_full python tools/profile_run.py --evals 2 > $OUT/ncu_full.log 2>&1
echo "ncu full rc=$?" >> $OUT/status.txt

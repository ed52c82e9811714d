#!/bin/bash
# GPU suite + smoke + the full default bench line.   bash tools/gpu_check.sh TAG
TAG=${1:-chk}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
( time timeout 1500 python bench.py ) > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt

#!/bin/bash
# Round-2 check on a cold box: smoke, the GPU parity suite (timed), the default bench.   bash tools/gpu_r2.sh TAG [bench args]
TAG=${1:-r2}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
( time timeout 300 python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 1100 python -m pytest tests -m gpu -q --durations=40 -p no:cacheprovider ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
if [ "${SKIP_BENCH:-0}" != "1" ]; then
  timeout 600 python bench.py "$@" > $OUT/bench.json 2> $OUT/bench.err
  echo "bench rc=$?" >> $OUT/status.txt
fi

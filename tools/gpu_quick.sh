#!/bin/bash
# Quick GPU iteration: parity tests + variant timings + bench.  bash tools/gpu_quick.sh TAG [variants]
TAG=${1:-q}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python tools/variants.py 1000 "${2:-vec=0}" > $OUT/variants.log 2>&1
echo "variants rc=$?" >> $OUT/status.txt
timeout 1200 python bench.py --steps 20 --warmup 5 ${BENCH_ARGS} > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt

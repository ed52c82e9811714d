#!/bin/bash
# GPU suite + window variants + the full default bench (all five configs).   bash tools/gpu_r2b.sh TAG
TAG=${1:-r2b}; OUT=gpurun_out/$TAG; mkdir -p $OUT
( time timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt
( time timeout 1500 python bench.py ) > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt

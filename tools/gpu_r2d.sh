#!/bin/bash
# GPU suite + ncu full profiles of the window kernel, staged and not.   bash tools/gpu_r2d.sh TAG
TAG=${1:-r2d}; OUT=gpurun_out/$TAG; mkdir -p $OUT
( time timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgb_window -c 1 -o $OUT/win_staged python bench.py --only --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/ncu_staged.log 2>&1; echo "ncu staged rc=$?" >> $OUT/status.txt
SGB_STAGE_ROWS=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgb_window -c 1 -o $OUT/win_plain python bench.py --only --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/ncu_plain.log 2>&1; echo "ncu plain rc=$?" >> $OUT/status.txt

#!/bin/bash
TAG=${1:-r3g}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( timeout 900 python bench.py --config c4 --only --no-cpu-baseline ) > $OUT/c4.json 2> $OUT/c4.err; echo "c4 rc=$?" >> $OUT/status.txt
( SGB_CSR_WINDOW=1 timeout 900 python bench.py --config c4 --only --no-cpu-baseline ) > $OUT/c4_win.json 2> $OUT/c4_win.err; echo "c4 win rc=$?" >> $OUT/status.txt
( SGB_CSR_WINDOW=1 timeout 900 python bench.py --config c3 --only --no-cpu-baseline ) > $OUT/c3_win.json 2> $OUT/c3_win.err; echo "c3 win rc=$?" >> $OUT/status.txt

#!/bin/bash
# Confirmation pass after the C1 e2e / batch-workspace changes: smoke, the full GPU suite, C1 and C5 lines.
TAG=${1:-f2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 1500 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for C in c1 c5 c3 c4; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "bench $C rc=$?" >> $OUT/status.txt
done
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo "bench c2 rc=$?" >> $OUT/status.txt

#!/bin/bash
# Quick round check: smoke, GPU parity suite, bench lines for C2/C3/C4.   bash tools/gpu_round.sh TAG
TAG=${1:-rr}
OUT=gpurun_out/$TAG
mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
( time python -c "import __graft_entry__ as g; g.smoke()" ) > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/status.txt
( time timeout 1200 python -m pytest tests -m gpu -x -q ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 900 python bench.py > $OUT/bench_c2.json 2> $OUT/bench_c2.err
echo "bench c2 rc=$?" >> $OUT/status.txt
for C in ${CONFIGS:-c3 c4}; do
  timeout 900 python bench.py --config $C --steps 10 --warmup 3 > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  echo "bench $C rc=$?" >> $OUT/status.txt
done

#!/bin/bash
# CSR windows vs gather on the bench configs + the GPU suite.   bash tools/gpu_win.sh TAG
TAG=${1:-win}
OUT=gpurun_out/$TAG
mkdir -p $OUT
( time timeout 900 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
for W in 1 0; do
  SGB_CSR_WINDOW=$W timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 4 --no-cpu-baseline > $OUT/c2_win$W.json 2> $OUT/c2_win$W.err
  echo "c2 win=$W rc=$?" >> $OUT/status.txt
done
SGB_CSR_WINDOW=1 timeout 600 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > $OUT/c1_win1.json 2> $OUT/c1_win1.err
echo "c1 rc=$?" >> $OUT/status.txt
SGB_CSR_WINDOW=1 timeout 600 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > $OUT/c4_win1.json 2> $OUT/c4_win1.err
echo "c4 rc=$?" >> $OUT/status.txt
SGB_CSR_WINDOW=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:sgb_window -c 3 --csv python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/ncu_win.csv 2> $OUT/ncu_win.err
echo "ncu rc=$?" >> $OUT/status.txt

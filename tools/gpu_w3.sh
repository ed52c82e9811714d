#!/bin/bash
OUT=gpurun_out/w3; mkdir -p $OUT
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt
SGB_CSR_WINDOW=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:sgb_window -c 1 -o $OUT/win_full python bench.py --steps 2 --warmup 3 --e2e-steps 2 --no-cpu-baseline > $OUT/ncu.log 2>&1; echo "ncu rc=$?" >> $OUT/status.txt

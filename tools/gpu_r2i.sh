#!/bin/bash
# Bulk-fed window kernel: GPU parity (builder plans, smoke) + window variants on C2 + the C2 bench.
TAG=${1:-r2i}; OUT=gpurun_out/$TAG; mkdir -p $OUT
( time timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "builder or csr_mode or wave_by_wave" ) > $OUT/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> $OUT/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/status.txt
timeout 900 python tools/win_variants.py > $OUT/variants.log 2>&1; echo "variants rc=$?" >> $OUT/status.txt
( time timeout 900 python bench.py --only ) > $OUT/bench.json 2> $OUT/bench.err
echo "bench rc=$?" >> $OUT/status.txt

#!/bin/bash
TAG=${1:-r3w}; OUT=gpurun_out/$TAG; mkdir -p $OUT
export SGB_PLAN_CACHE=/tmp/sgb_plan_cache_$TAG
for N in default 0 1024 default 0; do
  if [ "$N" = "default" ]; then unset SGB_JIT_MIN_N; else export SGB_JIT_MIN_N=$N; fi
  timeout 900 python bench.py --only --no-cpu-baseline --steps 20 > $OUT/c2_$N.json 2> $OUT/c2_$N.err
  python -c "import json;d=json.loads(open('$OUT/c2_$N.json').read().strip().splitlines()[-1]);print('$N', round(d['ms_per_step'],4), d['config']['parity'], d['gpu_launches'], [(l['name'],round(l['ms'],4)) for l in d['launches']])" >> $OUT/summary.txt
done

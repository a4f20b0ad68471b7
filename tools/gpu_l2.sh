#!/bin/bash
cd "$(dirname "$0")/.."
for spec in "21 13,8" "22 13,9" "23 13,10" "24 13,6,5" "25 13,6,6" "26 13,7,6"; do
  set -- $spec
  BW_PLAN=$2 timeout 600 python bench.py --log2n $1 --steps 200 --warmup 10 --no-e2e --no-cpu > gpurun_out/bench_l2.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_l2.log').read().strip().splitlines()[-1]); print('$1 $2', round(d['ms_per_step']*1e3,2),'us', d['passes_ms'], d['passes_gbs'])"
done

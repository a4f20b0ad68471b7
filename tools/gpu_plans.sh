#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for plan in 13,10,9 13,9,10 14,9,9 14,10,8 13,5,5,9 13,7,6,6; do
  BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_p.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); print('$plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done

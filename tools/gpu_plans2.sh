#!/bin/bash
cd "$(dirname "$0")/.."
for plan in 13,8,8,3 13,3,8,8 13,8,3,8 13,8,5,6 14,9,9; do
  BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_p.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); print('$plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done

#!/bin/bash
cd "$(dirname "$0")/.."
for f in 0 120000 0; do
for plan in "32 13,42,41" "32 14,9,9" "30 13,41,8" "32 13,8,8,3"; do
  set -- $plan
  BW_SMEM_FLOOR=$f BW_PLAN=$2 timeout 600 python bench.py --log2n $1 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1 || tail -3 gpurun_out/bench_ab.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('floor$f $1 $2', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done; done

#!/bin/bash
cd "$(dirname "$0")/.."
for pol in default spread balance; do
for plan in 14,9,9 13,42,41 14,42,42; do
  n=32; [ $plan = 14,42,42 ] && n=34
  BW_CLUSTER_POLICY=$pol BW_PLAN=$plan timeout 600 python bench.py --log2n $n --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v.log').read().strip().splitlines()[-1]); print('$pol $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done; done

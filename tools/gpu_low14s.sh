#!/bin/bash
cd "$(dirname "$0")/.."
BW_LOW14=s timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_n or split or int32" 2>&1 | tail -2
for v in s c; do
for plan in "32 14,9,9" "34 14,42,42" "24 14,10" "30 14,8,8"; do
  set -- $plan
  BW_LOW14=$v BW_PLAN=$2 timeout 600 python bench.py --log2n $1 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1 || tail -3 gpurun_out/bench_ab.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('$v $1 $2', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done; done

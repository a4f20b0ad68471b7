#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_n or split" 2>&1 | tail -1
for v in v c v; do
for plan in "30 13,41,8" "28 13,8,7" "26 13,8,5" "32 13,8,8,3"; do
  set -- $plan
  BW_HIGH13=$v BW_PLAN=$2 timeout 600 python bench.py --log2n $1 --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1 || tail -3 gpurun_out/bench_ab.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('$v $1 $2', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done; done

#!/bin/bash
cd "$(dirname "$0")/.."
for v in default minb3; do
 for plan in 13,8,8,3 13,10,9; do
  if [ $v = default ]; then L=""; else L="$PWD/build_variants/$v.so"; fi
  BW_LIB_PATH=$L BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_p.log 2>&1 || tail -5 gpurun_out/bench_p.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); print('$v $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
 done
done

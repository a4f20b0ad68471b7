#!/bin/bash
# A/B of library variants on the same box: tools/gpu_ab.sh "plan1 plan2" variant1 variant2 ...
cd "$(dirname "$0")/.."
plans=$1; shift
for rep in 1 2; do
for v in "$@"; do
 for plan in $plans; do
  BW_LIB_PATH=$PWD/build_variants/$v.so BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1 || tail -3 gpurun_out/bench_ab.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('$rep $v $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
 done
done
done

#!/bin/bash
# One-pass-per-variant A/B on the same box: tools/gpu_ab1.sh "plans" variants...
cd "$(dirname "$0")/.."
plans=$1; shift
for v in "$@"; do
 for plan in $plans; do
  n=32; case $plan in 14,42,42) n=34;; esac
  BW_LIB_PATH=$PWD/build_variants/$v.so BW_PLAN=$plan timeout 600 python bench.py --log2n $n --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_ab.log 2>&1 || tail -3 gpurun_out/bench_ab.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_ab.log').read().strip().splitlines()[-1]); print('$v $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
 done
done

#!/bin/bash
# Plan sweep for configs 3 (n=30) and 5 (n=34): entries r|(q+1)<<4 force the cluster size.
cd "$(dirname "$0")/.."
run() {
  c=$1; plan=$2
  BW_PLAN=$plan timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_s.log 2>&1 || { tail -3 gpurun_out/bench_s.log; return; }
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_s.log').read().strip().splitlines()[-1]); print('c$c $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'], [(p['k'],p['r'],p['cluster']) for p in d['config']['passes']])"
}
run 3 ""
for p in 13,41,24 13,24,41 13,42,23 13,23,42 14,24,24 13,41,40; do run 3 $p; done
run 5 ""
for p in 14,42,42 15,42,41 15,41,42 15,26,41; do run 5 $p; done

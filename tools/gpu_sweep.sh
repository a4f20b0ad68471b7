#!/bin/bash
# Plan sweep: entries r|(q+1)<<4 force a cluster of 2^q CTAs (26=10q0 25=9q0 41=9q1 42=10q1 58=10q2 24=8q0 40=8q1)
cd "$(dirname "$0")/.."
run() {
  n=$1; plan=$2
  BW_PLAN=$plan timeout 600 python bench.py --log2n $n --steps 10 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_s.log 2>&1 || { tail -3 gpurun_out/bench_s.log; return; }
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_s.log').read().strip().splitlines()[-1]); print('$n $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
}
for p in 13,8,5 14,7,5 13,13 14,12; do run 26 $p; done
for p in 13,8,7 14,7,7 14,14 13,41,6 15,13; do run 28 $p; done
for p in 13,25,8 13,41,8 14,8,8 14,41,7 15,8,7; do run 30 $p; done
for p in 14,9,9 14,41,41 14,25,41 13,41,42 13,41,58 14,40,41; do run 32 $p; done
for p in 14,42,42 14,58,58 14,26,42 15,41,58 15,42,41 14,41,41,1; do run 34 $p; done

#!/bin/bash
cd "$(dirname "$0")/.."
run() {
  n=$1; plan=$2
  BW_PLAN=$plan timeout 600 python bench.py --log2n $n --steps 10 --warmup 2 --no-e2e --no-cpu > gpurun_out/bench_s.log 2>&1 || { tail -3 gpurun_out/bench_s.log; return; }
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_s.log').read().strip().splitlines()[-1]); print('$n $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
}
for p in 14,10 13,11; do run 24 $p; done
for p in 13,8,5 13,7,6 14,7,5; do run 26 $p; done
for p in 13,8,7 13,5,5,5 14,7,7; do run 28 $p; done
for p in 13,25,8 13,41,8 14,8,8 13,6,6,5; do run 30 $p; done
for p in 13,42,41 13,26,41 14,9,9 13,8,8,3 13,7,6,6; do run 32 $p; done
for p in 14,42,42 13,7,7,7 15,41,42 13,42,41,2; do run 34 $p; done

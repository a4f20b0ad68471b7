#!/bin/bash
# Plan A/B at n=32: the 10-stage pass on 2- vs 4-CTA clusters.
cd "$(dirname "$0")/.."
run() {
  n=$1; plan=$2
  BW_PLAN=$plan timeout 600 python bench.py --log2n $n --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_s.log 2>&1 || { tail -3 gpurun_out/bench_s.log; return; }
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_s.log').read().strip().splitlines()[-1]); print('$n $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
}
for r in 1 2; do
run 32 13,42,41
run 32 13,58,41
run 32 13,58,57
run 32 13,41,42
done

#!/bin/bash
# Narrow plan at n = 32 with two tiles per CTA / cluster on the high passes.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "int64 1" "narrow 1" "narrow 2"; do
  set -- $v
  BW_NARROW_TPC=$2 timeout 300 python bench.py --log2n 32 --steps 5 --warmup 3 --no-e2e --no-cpu --intermediates $1 > gpurun_out/tpc.log 2>&1
  python -c "import json; d=json.loads([l for l in open('gpurun_out/tpc.log') if l.startswith('{')][0]); print('$1 tpc=$2', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'], d['config'].get('narrow_fallbacks'))" 2>/dev/null || tail -2 gpurun_out/tpc.log
done

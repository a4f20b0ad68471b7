#!/bin/bash
# Narrow plan variants at n = 32 (L2::256B loads in the mapped passes).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "13,10,9 int64 1" "13,10,9 narrow 1" "14,10,8 narrow 2" "13,10,9 narrow 1"; do
  set -- $v
  BW_PLAN=$1 BW_NARROW_TPC=$3 timeout 300 python bench.py --log2n 32 --steps 5 --warmup 3 --no-e2e --no-cpu --intermediates $2 > gpurun_out/tpc.log 2>&1
  python -c "import json; d=json.loads([l for l in open('gpurun_out/tpc.log') if l.startswith('{')][0]); print('$1 $2 tpc=$3', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'], d['config'].get('narrow_fallbacks'))" 2>/dev/null || tail -2 gpurun_out/tpc.log
done

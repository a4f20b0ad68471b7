#!/bin/bash
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,pci.bus_id,clocks.max.sm,clocks.sm,temperature.gpu,power.draw --format=csv
for r in 1 2 3; do
for plan in 14,9,9 13,42,41 13,25,41; do
  BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v.log').read().strip().splitlines()[-1]); print('$r $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'], d['clocks']['sm_mhz'])"
done; done

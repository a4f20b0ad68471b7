#!/bin/bash
# Every BASELINE config through bench.py (1 GPU).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > gpurun_out/bench_c$c.log 2>&1; echo "config $c rc=$?"
  tail -1 gpurun_out/bench_c$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['n'], '%.4g pts/s'%d['value'], round(d['ms_per_step'],3),'ms', d['passes_gbs'], 'frac', round(d['roofline']['frac'],3), 'e2e', d.get('e2e',{}).get('value'), 'cpu', d.get('cpu_baseline',{}).get('value'), d.get('extraction',''))" || tail -5 gpurun_out/bench_c$c.log
done

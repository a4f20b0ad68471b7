#!/bin/bash
# Config 2 (n = 24, 128 MiB, near the L2 size): candidate plans timed by bench.py (L2 flushed between steps).
cd "$(dirname "$0")/.."
for plan in default 14,10 15,9 13,11 13,5,6 13,6,5 13,3,8 13,8,3 14,5,5 13,2,9; do
  if [ $plan = default ]; then unset BW_PLAN; else export BW_PLAN=$plan; fi
  timeout 300 python bench.py --config 2 --steps 20 --warmup 5 --no-e2e --no-cpu 2>/dev/null | grep "^{" | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$plan', round(d['ms_per_step']*1000,1), 'us', [ (q['kind'],q['r'],q['cluster']) for q in d['config']['passes']])" || echo "$plan failed"
done

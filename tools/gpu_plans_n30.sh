#!/bin/bash
# n = 30 candidate plans (resident 8 GiB, +-1 input), timed by bench.py.
cd "$(dirname "$0")/.."
for plan in default 13,9,8 13,10,7 13,8,9 13,7,10 14,8,8 14,9,7 14,10,6 13,9,8,0; do
  if [ $plan = default ]; then unset BW_PLAN; else export BW_PLAN=$plan; fi
  timeout 300 python bench.py --log2n 30 --steps 10 --warmup 3 --no-e2e --no-cpu 2>/dev/null | grep "^{" | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$plan', round(d['ms_per_step'],3), 'ms', d['passes_gbs'], [(q['r'],q['cluster']) for q in d['config']['passes']])" 2>/dev/null || echo "$plan n/a"
done

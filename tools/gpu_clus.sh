#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
grep -q "rc=0" gpurun_out/pytest_gpu.log || exit 1
for plan in 13,10,9 14,9,9 15,9,8 15,10,7 13,9,10 14,10,8 15,8,9; do
  BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_p.log 2>&1 || tail -3 gpurun_out/bench_p.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); print('$plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done

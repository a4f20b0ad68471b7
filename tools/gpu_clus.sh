#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -6 gpurun_out/pytest_gpu.log
grep -q "rc=0" gpurun_out/pytest_gpu.log || exit 1
for plan in 14,9,9 13,42,41 15,9,8 13,58,41 14,58,8; do
  BW_PLAN=$plan timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_p.log 2>&1 || tail -3 gpurun_out/bench_p.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_p.log').read().strip().splitlines()[-1]); print('$plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done

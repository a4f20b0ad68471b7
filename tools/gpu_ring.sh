#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_n or split" > gpurun_out/ring_test.log 2>&1; echo "default tests rc=$?"
BW_RING=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "every_n or split" > gpurun_out/ring_test3.log 2>&1; echo "ring3 tests rc=$?"; tail -3 gpurun_out/ring_test3.log
for ring in 0 2 3; do
for plan in 13,42,41 13,8,8,3; do
  BW_RING=$ring BW_PLAN=$plan timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_v.log 2>&1 || tail -3 gpurun_out/bench_v.log
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_v.log').read().strip().splitlines()[-1]); print('ring$ring $plan', round(d['ms_per_step'],3), d['passes_ms'], d['passes_gbs'])"
done; done

#!/bin/bash
# GPU-box check: parity tests, smoke, a short bench.  Output -> gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_large.py -q -m gpu > gpurun_out/pytest_gpu_large.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_large.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -15 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log; tail -8 gpurun_out/pytest_gpu_large.log; tail -3 gpurun_out/bench.log

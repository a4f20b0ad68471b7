#!/bin/bash
# Full GPU check: every gpu test, then every config's bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/cfg
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in 1 2 3 4 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg/bench_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/cfg/bench_c$c.log
done

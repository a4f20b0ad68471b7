#!/bin/bash
# e2e leg A/B: K = 20 consecutive signals with two and three device buffers, then the default bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/e2e
mkdir -p $O
timeout 900 python bench.py --no-cpu --steps 20 --warmup 3 > $O/bench_k20_b2.log 2>&1; echo "rc=$?" >> $O/bench_k20_b2.log
BW_BATCH_BUFFERS=3 timeout 900 python bench.py --no-cpu --steps 20 --warmup 3 > $O/bench_k20_b3.log 2>&1; echo "rc=$?" >> $O/bench_k20_b3.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python -m pytest -q -m gpu tests/test_bench.py > $O/pytest_bench.log 2>&1; echo "rc=$?" >> $O/pytest_bench.log

#!/bin/bash
# Full verification: every GPU test, smoke, the default bench line, config 5,
# the reference arm.
cd "$(dirname "$0")/.."
O=gpurun_out/r2v
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > $O/bench_c5.log 2>&1; echo "rc=$?" >> $O/bench_c5.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log

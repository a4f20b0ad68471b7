#!/bin/bash
# After the capture guard and the stress-driver additions: the compact GPU
# tests, the race-stress build over every kernel family (3 repetitions), and
# a short default bench.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_check3
mkdir -p $O
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_compact.py tests/test_gpu_race_stress.py > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
ITERS=3 bash tools/race_stress.sh > $O/race_stress.log 2>&1; echo "rc=$?" >> $O/race_stress.log
timeout 600 python bench.py --no-e2e > $O/bench_default_noe2e.log 2> $O/bench.err; echo "rc=$?" >> $O/bench.err

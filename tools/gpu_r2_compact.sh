#!/bin/bash
# The compact plan as the default (n = 30..32): its GPU tests, the bench
# tests, per-pass timings at n = 24..32, and the default bench line.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_compact
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_compact.py tests/test_bench.py > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for n in 32 31 30 29 28 27 26 25 24; do
  echo "== --config 4 --n $n" >> $O/passes.log
  timeout 600 python tools/compact_bench.py --config 4 --n $n --reps 3 >> $O/passes.log 2>&1; echo "rc=$?" >> $O/passes.log
done
timeout 900 python bench.py > $O/bench_default.log 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
timeout 900 python bench.py --intermediates int64 --no-e2e --no-cpu > $O/bench_int64.log 2> $O/bench_int64.err; echo "rc=$?" >> $O/bench_int64.err

#!/bin/bash
# The int32-engine compact plan (v2): GPU parity of the compact tests, then
# pass-by-pass timings against the int64 plan at n = 30, 31, 32 (config 4),
# the first pass on the int64 engine (BW_COMPACT_FIRST=0) and v1 beside it.
cd "$(dirname "$0")/.."
O=gpurun_out/w32
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.log 2>&1
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_compact.py > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for args in "--config 4" "--config 4 --n 31" "--config 4 --n 30" ; do
  echo "== $args" >> $O/bench.log
  timeout 600 python tools/compact_bench.py $args --reps 3 >> $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
done
echo "== FIRST=0 --config 4" >> $O/bench.log
BW_COMPACT_FIRST=0 timeout 600 python tools/compact_bench.py --config 4 --reps 3 >> $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
echo "== v1 --config 4" >> $O/bench.log
BW_COMPACT_V2=0 timeout 600 python tools/compact_bench.py --config 4 --reps 3 >> $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log

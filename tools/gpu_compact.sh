#!/bin/bash
# The compact in-place plan: GPU parity tests, then timings at n = 32
# (config 4) and n = 34 (config 5) for a few plan shapes.
cd "$(dirname "$0")/.."
O=gpurun_out/compact
mkdir -p $O
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_compact.py > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for args in "--config 4" "--config 4 --tpc 2" "--config 4 --rows 9,9 --w 14" "--config 4 --n 31" \
            "--config 5" "--config 5 --rows 9,9,2" "--config 5 --tpc 2"; do
  echo "== $args" >> $O/bench.log
  timeout 600 python tools/compact_bench.py $args --reps 3 >> $O/bench.log 2>&1; echo "rc=$?" >> $O/bench.log
done

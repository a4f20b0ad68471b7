#!/bin/bash
# k32_high with 7 / 6 rows (n = 29 / 28: 8 rows first on the int32 engine):
# the compact GPU tests, then pass timings at n = 27..30.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_rows67
mkdir -p $O
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_compact.py > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for n in 30 29 28 27; do
  echo "== --config 4 --n $n" >> $O/passes.log
  timeout 600 python tools/compact_bench.py --config 4 --n $n --reps 3 >> $O/passes.log 2>&1; echo "rc=$?" >> $O/passes.log
done

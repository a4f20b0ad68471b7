#!/bin/bash
# The compact plan at n = 33 / 34 (+-1 signals: 9 + 8 rows on the int32 engine,
# 2 / 3 rows in registers, the 14-bit low pass): GPU parity of the register-pass
# shapes, pass timings against the int64 plan, and a full-size fold spot check.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_n34
mkdir -p $O
timeout 1500 python -m pytest -x -q -m gpu tests/test_gpu_compact.py -k "register_passes or full_size" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
for n in 33 34; do
  echo "== --config 4 --n $n" >> $O/passes.log
  timeout 900 python tools/compact_bench.py --config 4 --n $n --reps 2 >> $O/passes.log 2>&1; echo "rc=$?" >> $O/passes.log
done

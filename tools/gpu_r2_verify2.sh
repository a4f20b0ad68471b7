#!/bin/bash
# Round-2 verification with the compact plan as the default (n = 26..32):
# every GPU test, smoke, the default bench line, the reference arm, configs 1-3.
cd "$(dirname "$0")/.."
O=gpurun_out/${OUT:-r02_verify2}
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.log 2>&1
timeout 3000 python -m pytest -q -m gpu tests > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python __graft_entry__.py > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
for c in 1 2 3; do
  timeout 600 python bench.py --config $c --no-e2e > $O/bench_c$c.log 2> $O/bench_c$c.err; echo "rc=$?" >> $O/bench_c$c.err
done
BW_COMPACT=0 timeout 600 python bench.py --config 3 --no-e2e --no-cpu > $O/bench_c3_int64.log 2> $O/bench_c3_int64.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.log 2> $O/bench_reference.err; echo "rc=$?" >> $O/bench_reference.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > $O/bench_c5.log 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err

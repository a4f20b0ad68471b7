#!/bin/bash
# End-of-session evidence: every GPU test, smoke, the default bench line
# (driver command), every config's bench line, and the n = 32 launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/final
timeout 1800 python -m pytest tests -q -m gpu > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py > gpurun_out/final/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench_reference.log
for c in 1 2 3 5; do
  timeout 900 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/final/bench_c$c.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench_c$c.log
done
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/final/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches_n32.csv $B \
    > gpurun_out/final/ncu_launch.log 2>&1; echo "launch rc=$?" >> gpurun_out/final/ncu_launch.log

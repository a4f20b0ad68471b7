#!/bin/bash
# Session check: every GPU test, smoke, the driver's default bench line, and
# ncu of the split-row kernel (n = 33 plan: 13 + split 10 + 10).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
P="python tools/prof_passes.py --n 33 --reps 1"
$P > gpurun_out/plain_prof33.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_n33.csv $P > gpurun_out/ncu_launch33.log 2>&1
echo "launch rc=$?" >> gpurun_out/ncu_launch33.log
ncu --set full --clock-control none --import-source on -k regex:k_pass_split -c 1 -o gpurun_out/prof_n33_split $P \
    > gpurun_out/ncu_full33.log 2>&1
echo "full rc=$?" >> gpurun_out/ncu_full33.log

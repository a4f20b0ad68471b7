#!/bin/bash
# Round evidence: (1) the default bench line, (2) the launch list of the same
# command (gpu__time_duration per launch), (3) ncu --set full on the three
# passes of one n=32 transform (profiling driver, same kernels and plan).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$B > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_final.csv $B > gpurun_out/ncu_launch.log 2>&1
echo "launch rc=$?"
P="python tools/prof_passes.py --n 32 --reps 2"
$P > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 3 -o gpurun_out/prof_n32_final $P \
    > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full.log

#!/bin/bash
cd "$(dirname "$0")/.."
P="python tools/prof_passes.py --n 28 --reps 2"
BW_PLAN=14,58,4 $P > gpurun_out/plain_prof.log 2>&1 && \
BW_PLAN=14,58,4 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 2 -o gpurun_out/prof_q2 $P > gpurun_out/ncu_full.log 2>&1
echo "q2 rc=$?"
BW_PLAN=13,41,6 $P > gpurun_out/plain_prof.log 2>&1 && \
BW_PLAN=13,41,6 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 4 -c 1 -o gpurun_out/prof_q1 $P > gpurun_out/ncu_full2.log 2>&1
echo "q1 rc=$?"

#!/bin/bash
cd "$(dirname "$0")/.."
P="python tools/prof_passes.py --n 26 --reps 2"
export BW_PLAN=15,10,1
$P > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 2 -o gpurun_out/prof_clus2 $P > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full.log

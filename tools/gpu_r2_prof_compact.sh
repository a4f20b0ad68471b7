#!/bin/bash
# ncu evidence for the compact plan (the default at n = 26..32): the launch
# list of the default bench command, and ncu --set full of one n = 32
# transform's three kernels (k32_first checked, k32_high, k32_low), summarised
# on the box (the .ncu-rep is too large to bring back).
cd "$(dirname "$0")/.."
O=gpurun_out/r02_prof_compact
mkdir -p $O
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 600 $B > $O/bench_short.log 2>&1; echo "rc=$?" >> $O/bench_short.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_n32.csv $B > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
timeout 300 python tools/prof_passes.py --n 32 --reps 2 > $O/prof_passes.log 2>&1; echo "rc=$?" >> $O/prof_passes.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:k32_ -s 3 -c 3 -o /tmp/prof_c32 \
    python tools/prof_passes.py --n 32 --reps 2 > $O/ncu_full_n32.log 2>&1; echo "rc=$?" >> $O/ncu_full_n32.log
python tools/ncu_summary.py /tmp/prof_c32.ncu-rep $O/r02_n32_compact 32 > $O/ncu_summary_n32.log 2>&1
gzip -f $O/r02_n32_compact_source.csv
du -sh $O

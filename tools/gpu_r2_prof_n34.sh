#!/bin/bash
# ncu --set full of one n = 34 transform on the compact plan (k32_first checked, k32_high<6>, k32_reg<3>, k32_low),
# summarised on the box.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_prof_n34
mkdir -p $O
timeout 600 python tools/prof_passes.py --n 34 --reps 2 > $O/prof_passes.log 2>&1; echo "rc=$?" >> $O/prof_passes.log
timeout 2400 ncu --set full --clock-control none --import-source on -f -k regex:k32_ -s 6 -c 4 -o /tmp/prof_c34 \
    python tools/prof_passes.py --n 34 --reps 2 > $O/ncu_full_n34.log 2>&1; echo "rc=$?" >> $O/ncu_full_n34.log
python tools/ncu_summary.py /tmp/prof_c34.ncu-rep $O/r02_n34_compact 34 > $O/ncu_summary_n34.log 2>&1
gzip -f $O/r02_n34_compact_source.csv

#!/bin/bash
# Round-2 evidence after the split-kernel change: every GPU test, smoke, the
# default bench line (n = 32) and config 5 (n = 34), the launch list of the
# default bench, and ncu --set full of one n = 32 and one n = 34 transform
# (summarised on the box; the .ncu-rep files are too large to bring back).
cd "$(dirname "$0")/.."
O=gpurun_out/r2f
mkdir -p $O
timeout 2400 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > $O/bench_c5.log 2>&1; echo "rc=$?" >> $O/bench_c5.log
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $O/launches_n32.csv $B > $O/ncu_launch.log 2>&1; echo "rc=$?" >> $O/ncu_launch.log
for n in 32 34; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 3 -c 3 -o /tmp/prof_n$n \
      python tools/prof_passes.py --n $n --reps 2 > $O/ncu_full_n$n.log 2>&1; echo "rc=$?" >> $O/ncu_full_n$n.log
  python tools/ncu_summary.py /tmp/prof_n$n.ncu-rep $O/r02_n$n $n > $O/ncu_summary_n$n.log 2>&1
done
du -sh $O
ITERS=3 bash tools/race_stress.sh

#!/bin/bash
# Per-step input regeneration A/B on one box, and split-row plan sweeps at n = 28..31.
cd "$(dirname "$0")/.."
O=gpurun_out/restore
mkdir -p $O
for i in 1 2; do
  timeout 600 python bench.py --no-cpu --no-e2e --no-entry-points > $O/bench_restore_$i.log 2>&1
  BW_BENCH_RESTORE=0 timeout 600 python bench.py --no-cpu --no-e2e --no-entry-points > $O/bench_b2b_$i.log 2>&1
done
for n in 28 30 31; do
  timeout 600 python tools/sweep_split.py --n $n --out $O/split_n$n.json > $O/split_n$n.log 2>&1
done

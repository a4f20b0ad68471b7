#!/bin/bash
# How the input is restored between steps: the generator vs a device copy vs none.
cd "$(dirname "$0")/.."
O=gpurun_out/restore2
mkdir -p $O
for i in 1 2; do
  for m in 1 copy 0; do
    BW_BENCH_RESTORE=$m timeout 600 python bench.py --no-cpu --no-e2e --no-entry-points > $O/bench_${m}_$i.log 2>&1
  done
done

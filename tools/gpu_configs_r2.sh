#!/bin/bash
# Configs 1-3 with the round-2 library (config 4 and 5 are in r02_verify).
cd "$(dirname "$0")/.."
O=gpurun_out/configs_r2
mkdir -p $O
for c in 1 2 3; do
  timeout 900 python bench.py --config $c > $O/bench_c$c.log 2>&1; echo "rc=$?" >> $O/bench_c$c.log
done

#!/bin/bash
# A/B of the low passes' L2 bulk prefetch distance (BW_LOW_PREFETCH, tiles):
# n = 34 (14-bit low pass on 2-CTA clusters) and n = 32 (13-bit, one CTA).
cd "$(dirname "$0")/.."
O=gpurun_out/prefetch
mkdir -p $O
for d in 0 37 74 148 296 592 0; do
  for n in 34 32; do
    echo "== n=$n BW_LOW_PREFETCH=$d" >> $O/ab.log
    BW_LOW_PREFETCH=$d timeout 300 python tools/pass_data_study.py --n $n --reps 2 --kinds zeros,pm1 2>&1 | grep -v "^{" >> $O/ab.log
  done
done
timeout 900 python -m pytest -q -m gpu tests -k "extract or xfused or fused or config3 or config5" > $O/pytest_extract.log 2>&1; echo "rc=$?" >> $O/pytest_extract.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_c5.log 2>&1; echo "rc=$?" >> $O/bench_c5.log

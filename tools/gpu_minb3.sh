#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/minb3
mkdir -p $O
BW_LOW14_MINB3=1 timeout 300 python tools/sanitize_driver.py --family cluster > $O/parity.log 2>&1; echo "rc=$?" >> $O/parity.log
for v in 0 1 0 1; do
  echo "== BW_LOW14_MINB3=$v" >> $O/ab.log
  BW_LOW14_MINB3=$v timeout 300 python tools/pass_data_study.py --n 34 --reps 2 --kinds zeros,noisy 2>&1 | grep -v "^{" >> $O/ab.log
done

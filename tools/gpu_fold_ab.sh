#!/bin/bash
# Block-fold shape A/B (bins per CTA, threads per CTA) on the same box.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in fold_13_512 fold_12_256 fold_12_512 fold_13_256; do
  if [ $v = default ]; then L=""; else L=$PWD/build_variants/$v.so; fi
  echo "== $v"
  BW_LIB_PATH=$L timeout 300 python tools/fold_bench.py 32 2>&1 | grep -v "n=34"
done

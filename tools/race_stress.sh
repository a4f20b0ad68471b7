#!/bin/bash
# Dynamic race check (compute-sanitizer is closed on this pool): every kernel
# family of tools/sanitize_driver.py, ITERS times, against the race-stress
# build (-DBW_RACE_STRESS: random warp sleeps at every synchronisation point,
# python -m paper_1607_01039_b200.build --stress), each result compared with
# the CPU oracle.  Logs under gpurun_out/race_stress/.
cd "$(dirname "$0")/.."
O=gpurun_out/race_stress
mkdir -p $O
ITERS=${ITERS:-5}
export BW_LIB_PATH=$PWD/paper_1607_01039_b200/lib/libbigwht_b200_stress.so
for i in $(seq 1 $ITERS); do
  timeout 900 python tools/sanitize_driver.py > $O/iter$i.log 2>&1; echo "rc=$?" >> $O/iter$i.log
done
BW_NARROW_TPC=1 timeout 600 python tools/sanitize_driver.py --family map > $O/map_tpc1.log 2>&1; echo "rc=$?" >> $O/map_tpc1.log
grep -H "MISMATCH\|rc=" $O/*.log > $O/summary.txt

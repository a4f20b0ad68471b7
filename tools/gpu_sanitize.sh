#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck on one small invocation
# of every kernel family (tools/sanitize_driver.py), logs under
# gpurun_out/sanitize/.  Each run is bounded by its own timeout.
cd "$(dirname "$0")/.."
O=gpurun_out/sanitize
mkdir -p $O
python tools/sanitize_driver.py > $O/plain.log 2>&1; echo "plain rc=$?" >> $O/plain.log
for fam in low1 cluster split two_pass map xfused narrow extract fold aux; do
  for tool in memcheck racecheck synccheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 600 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
        python tools/sanitize_driver.py --family $fam > $O/${tool}_${fam}.log 2>&1
    echo "rc=$?" >> $O/${tool}_${fam}.log
  done
done
# the 2-CTA narrow map with one tile per cluster, too
BW_NARROW_TPC=1 timeout 600 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_driver.py --family map > $O/racecheck_map_tpc1.log 2>&1; echo "rc=$?" >> $O/racecheck_map_tpc1.log
grep -H "ERROR SUMMARY\|RACECHECK SUMMARY\|rc=" $O/*.log > $O/summary.txt

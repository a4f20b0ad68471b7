#!/bin/bash
# fwht_inplace with the fused bound check: its tests, the race-stress run of
# every family (bound included), and the bench line (entry_points).
cd "$(dirname "$0")/.."
O=gpurun_out/bound
mkdir -p $O
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_fused_bound.py tests/test_gpu_race_stress.py tests/test_gpu_parity.py -k "bound or overflow or stress or inplace" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
BW_FUSED_BOUND=0 timeout 900 python bench.py --no-e2e --no-cpu > $O/bench_nofused.log 2>&1; echo "rc=$?" >> $O/bench_nofused.log

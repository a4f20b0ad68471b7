#!/bin/bash
# fwht_arrays with the per-signal copy pipeline: its tests, then the e2e leg A/B.
cd "$(dirname "$0")/.."
O=gpurun_out/batch
mkdir -p $O
timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py -k "host_batch or host_buffer" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
timeout 900 python bench.py --no-cpu > $O/bench_pipe.log 2>&1; echo "rc=$?" >> $O/bench_pipe.log
BW_BATCH_PIPELINE=0 timeout 900 python bench.py --no-cpu > $O/bench_nopipe.log 2>&1; echo "rc=$?" >> $O/bench_nopipe.log

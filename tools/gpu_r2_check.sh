#!/bin/bash
# Round-2 check: the new boundary / bench-parity tests first, then every GPU
# test, smoke, the driver's default bench line and the reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 900 python -m pytest -q -m gpu tests/test_reference_suite.py tests/test_bench.py \
    "tests/test_gpu_parity.py::test_host_batch_reused_buffers_any_work_count" > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 1800 python -m pytest tests -q -m gpu > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.log 2>&1; echo "rc=$?" >> $O/bench_default.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.log 2>&1; echo "rc=$?" >> $O/bench_reference.log

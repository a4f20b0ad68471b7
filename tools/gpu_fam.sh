#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
for f in 14 13; do
  BW_LOW_BITS=$f timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_f$f.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_f$f.log').read().strip().splitlines()[-1]); print($f, d['ms_per_step'], d['passes_ms'], d['passes_gbs'], d['clocks'])"
done
for n in 30 28; do
BW_LOW_BITS=13 timeout 600 python bench.py --log2n $n --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_n$n.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_n$n.log').read().strip().splitlines()[-1]); print($n, d['ms_per_step'], d['passes_ms'], d['passes_gbs'])"
done

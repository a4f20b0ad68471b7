#!/bin/bash
# n = 33 / 34 on the compact plan as the default: the compact GPU tests (register-pass shapes, full-size
# spot checks up to n = 34), the n = 34 tests of the large suite (config 5 goes through the sample
# refusal), config 5's bench and a +-1 bench line at n = 34.
cd "$(dirname "$0")/.."
O=gpurun_out/r02_n34b
mkdir -p $O
timeout 1800 python -m pytest -x -q -m gpu tests/test_gpu_compact.py -k "register_passes or full_size or default" --durations=5 > $O/pytest_compact.log 2>&1; echo "rc=$?" >> $O/pytest_compact.log
timeout 1800 python -m pytest -x -q -m gpu tests/test_gpu_large.py --durations=5 > $O/pytest_large.log 2>&1; echo "rc=$?" >> $O/pytest_large.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > $O/bench_c5.log 2> $O/bench_c5.err; echo "rc=$?" >> $O/bench_c5.err
timeout 900 python bench.py --config 4 --log2n 34 --steps 5 --warmup 3 --no-e2e > $O/bench_pm1_n34.log 2> $O/bench_pm1_n34.err; echo "rc=$?" >> $O/bench_pm1_n34.err
timeout 900 python bench.py --config 4 --log2n 33 --steps 5 --warmup 3 --no-e2e --no-cpu > $O/bench_pm1_n33.log 2> $O/bench_pm1_n33.err; echo "rc=$?" >> $O/bench_pm1_n33.err
timeout 600 python tools/refused_bench.py --n 34 --reps 2 > $O/refused_n34.log 2>&1; echo "rc=$?" >> $O/refused_n34.log

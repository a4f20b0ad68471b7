#!/bin/bash
# Round-2 evidence: per-pass rate vs the data in the signal (n = 34), the
# split walk on zero vs random data, one full-size run of the reference's
# run_parallel (n = 32) next to the extrapolated samples, config 5, then the
# compute-sanitizer runs.
cd "$(dirname "$0")/.."
O=gpurun_out/r2e
mkdir -p $O
timeout 600 python tools/pass_data_study.py --n 34 --reps 2 > $O/data_study_n34.log 2>&1; echo "rc=$?" >> $O/data_study_n34.log
timeout 300 tools/bin/mb_split > $O/mb_split_zeros.log 2>&1; echo "rc=$?" >> $O/mb_split_zeros.log
timeout 300 tools/bin/mb_split rand > $O/mb_split_rand.log 2>&1; echo "rc=$?" >> $O/mb_split_rand.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e > $O/bench_c5.log 2>&1; echo "rc=$?" >> $O/bench_c5.log
timeout 1200 python bench.py --cpu-full --no-e2e --steps 5 --warmup 3 > $O/bench_cpu_full.log 2>&1; echo "rc=$?" >> $O/bench_cpu_full.log
cp profiles/r02_cpu_reference_full.json $O/ 2>/dev/null
bash tools/gpu_sanitize.sh

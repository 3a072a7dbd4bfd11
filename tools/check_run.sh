#!/bin/bash
# Bounds-checked build (make check) over the GPU parity tests, every engine's small cases
# (tools/sanitize_run.py) and two bench workloads; logs under gpurun_out/$1/.
set -u
O=gpurun_out/${1:-check}; mkdir -p $O
export GLS_LIB=$PWD/paper_2304_13398_b200/libgls_check.so
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 --deselect tests/test_gpu_fullsize.py::test_c5_all_sets > $O/pytest_gpu_check.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu_check.log
timeout 600 python tools/sanitize_run.py 40 > $O/small_cases_check.log 2>&1; echo "rc=$?" >> $O/small_cases_check.log
timeout 600 python bench.py --config c4_mini --steps 1 --warmup 1 --no-e2e > $O/bench_c4mini_check.json 2> $O/bench_c4mini_check.log; echo "rc=$?" >> $O/bench_c4mini_check.log
timeout 600 python bench.py --config c5_set --steps 1 --warmup 1 --no-e2e > $O/bench_c5_check.json 2> $O/bench_c5_check.log; echo "rc=$?" >> $O/bench_c5_check.log
grep -h "GLS_CHECK\|passed\|failed\|rc=\|mismatch" $O/*.log | head -20

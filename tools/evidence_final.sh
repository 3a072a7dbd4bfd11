#!/bin/bash
# Final check of a commit on one B200: bench (C4 default, C3), GPU tests, smoke.
set -u
O=gpurun_out/${1:-final}; mkdir -p $O
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.log
timeout 600 python bench.py --config c3_1m > $O/bench_c3.json 2> $O/bench_c3.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log

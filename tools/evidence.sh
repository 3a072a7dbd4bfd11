#!/bin/bash
# Round evidence on one B200: GPU tests, smoke, default bench, reference arm, ncu launch list.
# usage: tools/evidence.sh TAG   (outputs under gpurun_out/TAG/)
set -u
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.log
# launch list of the bench command (serialised, cold-cache; shares, not absolutes) + DRAM bytes per launch
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
tail -c 3000 $O/bench.json $O/bench_ref.json $O/smoke.log $O/pytest_gpu.log
# one full ncu capture of the kernel on the c4_mini workload (source-level stalls)
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/c4mini_full \
  python bench.py --config c4_mini --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1

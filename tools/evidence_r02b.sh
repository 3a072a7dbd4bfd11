#!/bin/bash
# Round-2 final evidence on one B200: GPU tests, smoke, benches, reference arm, launch list,
# one full ncu capture of sim_kernel on c4_mini.  Outputs under gpurun_out/TAG/.
set -u
TAG=${1:-r02b}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $O/nproc.txt
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.log
timeout 600 python bench.py --config c3_1m > $O/bench_c3.json 2> $O/bench_c3.log
timeout 900 python bench.py --config c5_set --steps 2 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.log
timeout 300 python bench.py --config c7552 > $O/bench_c7552.json 2> $O/bench_c7552.log
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/c4mini_full \
  python bench.py --config c4_mini --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
tail -c 1500 $O/bench_c4.json; tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log

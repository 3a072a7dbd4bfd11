set -u
O=gpurun_out/r02a; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > $O/gpu.txt 2>&1
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.log
timeout 600 python bench.py --config c3_1m --no-e2e > $O/bench_c3.json 2> $O/bench_c3.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_bench.log 2>&1
tail -c 1500 $O/bench_c4.json $O/bench_c3.json; tail -5 $O/bench_c4.log

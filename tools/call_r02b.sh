set -u
O=gpurun_out/r02c; mkdir -p $O
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cells.py -m gpu -x -q -k "auto" --timeout 90 > $O/pytest_auto.log 2>&1; echo "rc=$?" >> $O/pytest_auto.log
tail -15 $O/pytest_auto.log
timeout 150 python bench.py --engine 3 --config c3_1m --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > $O/c3_e3.json 2> $O/c3_e3.log
tail -3 $O/c3_e3.log
timeout 200 python bench.py --engine 3 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > $O/c4_e3.json 2> $O/c4_e3.log
tail -4 $O/c4_e3.log

set -u
T=r02i; O=gpurun_out/$T; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cells.py -m gpu -x -q -k "auto" --timeout 60 > $O/pytest_auto.log 2>&1; echo "rc=$?" >> $O/pytest_auto.log
tail -3 $O/pytest_auto.log
export EXTRA="--engine 3"
bash tools/ab2.sh $T "default r8 r2" "c3_1m c4_10m"
EXTRA="--engine 3 --chunk-events 512" SUF=_m512 bash tools/ab2.sh $T "default r8" "c3_1m c4_10m"

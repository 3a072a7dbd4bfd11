set -u
T=r02t
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cells.py -m gpu -x -q --timeout 120 > gpurun_out/$T.pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/$T.pytest.log
export EXTRA=""
bash tools/ab2.sh $T "default d0 d32k" "c4_10m c3_1m c5_set"
bash tools/ab2.sh ${T}b "default d0" "c4_10m c3_1m"

set -u
T=r02j; O=gpurun_out/$T; mkdir -p $O
for e in 3 0; do
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/e${e}_c3s \
  python bench.py --engine $e --config c3_1m --ncycles 2000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_e$e.log 2>&1
tail -1 $O/ncu_e$e.log
done

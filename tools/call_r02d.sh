set -u
T=r02d
export EXTRA="--engine 3"
bash tools/ab2.sh $T "default pf2 pf4 noacq r64" "c3_1m c4_10m"
EXTRA="--engine 3 --chunk-events 512" SUF=_m512 bash tools/ab2.sh $T "default pf2" "c3_1m c4_10m"
EXTRA="--engine 3 --chunk-events 1024" SUF=_m1k bash tools/ab2.sh $T "default" "c4_10m"
O=gpurun_out/$T
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/e3_c4mini \
  python bench.py --engine 3 --config c4_mini --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_e3.log 2>&1
tail -2 $O/ncu_e3.log

set -u
T=r02p; O=gpurun_out/$T; mkdir -p $O
EXTRA="--chunk-events 65536" SUF=_m64k bash tools/ab2.sh $T "default" "c4_10m c3_1m c5_set"
EXTRA="--chunk-events 131072" SUF=_m128k bash tools/ab2.sh $T "default" "c4_10m c3_1m"
EXTRA="--chunk-events 32768" SUF=_m32k bash tools/ab2.sh $T "default" "c5_set"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/c4mini_full \
  python bench.py --config c4_mini --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_full.log 2>&1
tail -1 $O/ncu_full.log

timeout 900 python tools/wcv_sweep.py 60000 > $O/wcv_sweep.jsonl 2> $O/wcv_sweep.log
cat $O/wcv_sweep.jsonl

set -u
T=r02r; O=gpurun_out/$T; mkdir -p $O
timeout 900 python tools/wcv_sweep.py > $O/wcv_sweep_full.jsonl 2> $O/wcv_sweep_full.log
timeout 600 python tools/wcv_sweep.py 60000 > $O/wcv_sweep_60k.jsonl 2> $O/wcv_sweep_60k.log
cat $O/wcv_sweep_full.jsonl $O/wcv_sweep_60k.jsonl
bash tools/sanitize.sh $T/sanitize

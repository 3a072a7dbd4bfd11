#!/bin/bash
# Functional run of bench.py's N > 1 code paths (time windows + both stitches; stimulus-set
# replicas + the per-set checksum all_gather; the reference arm) with 2 ranks on ONE GPU:
# gloo collectives staged through host memory, every rank on cuda:0, explicit arenas.  Not a
# measurement (the ranks share one GPU); the product runs one rank per GPU over NCCL.
set -u
O=gpurun_out/${1:-multirank}; mkdir -p $O
export GLS_BENCH_BACKEND=gloo GLS_BENCH_ONE_GPU=1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 900 $TR bench.py --gpus 2 --config c3_1m --ncycles 2000 --arena-gb 24 --steps 2 --warmup 3 --no-e2e \
  > $O/c3_2ranks.json 2> $O/c3_2ranks.log; echo "c3 windows rc=$?"
GLS_BENCH_C5_SETS=4 timeout 900 $TR bench.py --gpus 2 --config c5_set --arena-gb 24 --steps 1 --warmup 3 --no-e2e \
  > $O/c5_2ranks.json 2> $O/c5_2ranks.log; echo "c5 sets rc=$?"
timeout 600 $TR bench.py --gpus 2 --impl reference --config c7552 --steps 1 --warmup 3 > $O/ref_2ranks.json 2> $O/ref_2ranks.log; echo "ref rc=$?"
for f in c3_2ranks c5_2ranks ref_2ranks; do echo "== $f"; tail -c 1500 $O/$f.json; done

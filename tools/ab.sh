#!/bin/bash
# A/B of library variants on the default bench workload: tools/ab.sh TAG variant...
# (variant "default" = paper_2304_13398_b200/libgls.so, else paper_2304_13398_b200/libgls_<v>.so)
TAG=$1; shift
O=gpurun_out/$TAG; mkdir -p $O
for v in "$@"; do
  if [ "$v" = default ]; then unset GLS_LIB; else export GLS_LIB=$PWD/paper_2304_13398_b200/libgls_$v.so; fi
  timeout 600 python bench.py --steps 2 --warmup 2 --no-cpu-baseline --no-e2e ${BENCH_ARGS:-} > $O/bench_$v.json 2> $O/bench_$v.log
  echo "== $v"; tail -1 $O/bench_$v.log | cut -c1-330
done

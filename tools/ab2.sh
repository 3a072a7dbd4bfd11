#!/bin/bash
# A/B of library variants on bench configs: tools/ab2.sh TAG "variants" "configs"
# (variant "default" = libgls.so, else libgls_<v>.so); prints the last warm-up line per run
TAG=$1; O=gpurun_out/$TAG; mkdir -p $O
for v in $2; do for c in $3; do
  if [ "$v" = default ]; then unset GLS_LIB; else export GLS_LIB=$PWD/paper_2304_13398_b200/libgls_$v.so; fi
  if [ "$v" = old ]; then export GLS_AB_OLD=1; else unset GLS_AB_OLD; fi
  timeout 400 python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e $EXTRA > $O/${v}_$c${SUF}.json 2> $O/${v}_$c${SUF}.log
  echo "== $v $c: $(grep "warmup 1" $O/${v}_$c${SUF}.log | sed -E 's/, [0-9]+ gate-evals, [0-9]+ outputs//' | cut -c1-330)"
done; done

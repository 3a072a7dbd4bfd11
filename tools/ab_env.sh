#!/bin/bash
# A/B with env settings: tools/ab_env.sh "LIB:ENV=VAL LIB2:ENV=VAL" "cfg..."   (ENV part optional, e.g. libgls:GLS_CARVEOUT=-1)
for spec in $1; do L=${spec%%:*}; E=""; [ "$spec" != "$L" ] && E=${spec#*:}; for c in $2; do
  env GLS_LIB=paper_2304_13398_b200/$L.so $E timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 \
    | grep "warmup 2" | sed -E 's/, [0-9]+ gate-evals, [0-9]+ outputs, [0-9]+ chunks//' | cut -c1-200 | sed "s/^\[bench\] warmup 2:/$spec $c/"
done; done

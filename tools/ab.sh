#!/bin/bash
# A/B timing of library variants: tools/ab.sh "libA libB ..." "cfg1 cfg2 ..."
for L in $1; do for c in $2; do
  GLS_LIB=paper_2304_13398_b200/$L.so timeout 300 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 \
    | grep "warmup 2" | sed -E 's/, [0-9]+ gate-evals, [0-9]+ outputs, [0-9]+ chunks//' | cut -c1-260 | sed "s/^\[bench\] warmup 2:/$L $c/"
done; done

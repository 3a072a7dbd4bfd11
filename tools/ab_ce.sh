#!/bin/bash
# chunk-size sweep: tools/ab_ce.sh TAG "chunk_events values" "configs"
TAG=$1; O=gpurun_out/$TAG; mkdir -p $O
for m in $2; do for c in $3; do
  timeout 400 python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline --no-e2e --chunk-events $m > $O/ce${m}_$c.json 2> $O/ce${m}_$c.log
  echo "== M=$m $c: $(grep 'warmup 1' $O/ce${m}_$c.log | sed -E 's/, [0-9]+ gate-evals, [0-9]+ outputs//' | cut -c1-330)"
done; done

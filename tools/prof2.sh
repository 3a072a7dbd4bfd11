#!/bin/bash
# full ncu capture of sim_kernel for library variants on one config: tools/prof2.sh TAG CONFIG "variants"
TAG=$1; CFG=$2; O=gpurun_out/$TAG; mkdir -p $O
for v in $3; do
  if [ "$v" = default ]; then unset GLS_LIB; else export GLS_LIB=$PWD/paper_2304_13398_b200/libgls_$v.so; fi
  case $v in old*) export GLS_AB_OLD=1;; *) unset GLS_AB_OLD;; esac
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:sim_kernel -s 1 -c 1 -o $O/${v}_$CFG \
    python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e $EXTRA > $O/ncu_${v}.log 2>&1
  echo "== $v: $(tail -1 $O/ncu_${v}.log)"
done

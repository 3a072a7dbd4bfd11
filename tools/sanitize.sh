#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck, synccheck, initcheck
# (logs under gpurun_out/$1/); usage: tools/sanitize.sh TAG
O=gpurun_out/${1:-sanitize}; mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  n=40; [ $tool = racecheck ] && n=8; [ $tool = initcheck ] && n=20
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 --target-processes all \
    python tools/sanitize_run.py $n > $O/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' $O/$tool.log | tr '\n' ' ')"
done

#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck, synccheck, initcheck
# (logs under gpurun_out/$1/); usage: tools/sanitize.sh TAG
O=gpurun_out/${1:-sanitize}; mkdir -p $O
for tool in memcheck racecheck synccheck initcheck; do
  n=16; [ $tool = racecheck ] && n=3; [ $tool = initcheck ] && n=6; [ $tool = synccheck ] && n=6
  timeout 700 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 3 --target-processes all \
    python tools/sanitize_run.py $n > $O/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run' $O/$tool.log | tr '\n' ' ')"
done

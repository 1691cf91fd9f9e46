#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every execution tier
# (tools/sanitize_cases.py):  bash tools/gpu_sanitize.sh <tag> [cases...]
tag=${1:-san}; shift; out=gpurun_out/$tag; mkdir -p $out
cases=${@:-tiles cluster fused graded lu nograph dist}
for tool in memcheck racecheck synccheck; do
  for c in $cases; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check no"
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 20 \
        python tools/sanitize_cases.py $c > $out/${tool}_$c.log 2>&1
    echo "$tool $c exit $? $(grep -c '========= ' $out/${tool}_$c.log) sanitizer lines; $(grep 'ERROR SUMMARY\|RACECHECK SUMMARY' $out/${tool}_$c.log | tail -1)" >> $out/summary.txt
  done
done
cat $out/summary.txt

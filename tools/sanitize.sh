#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the small cases of tools/sanitize.py
# (VERDICT r01 #8).  Logs: gpurun_out/sanitize_<tag>_<tool>_<case>.log; summary on stdout.
TAG=${1:-r02}
CASES=${CASES:-"c0 c1s c2 c3 c4 m1 s1"}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for c in $CASES; do
    log=gpurun_out/sanitize_${TAG}_${tool}_${c}.log
    extra=""
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 99 --target-processes all \
      python tools/sanitize.py $c > $log 2>&1
    rc=$?
    echo "$tool $c rc=$rc $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' $log | tail -1)"
  done
done

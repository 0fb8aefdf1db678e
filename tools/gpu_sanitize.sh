#!/bin/bash
# compute-sanitizer over every device code path (tools/sanitize_cases.py).
TAG=${1:-san}; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
python tools/sanitize_cases.py > $OUT/plain.log 2>&1; echo "plain rc=$?" >> $OUT/plain.log
for tool in memcheck initcheck synccheck racecheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 python tools/sanitize_cases.py "$@" > $OUT/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $OUT/sanitize_$tool.log
done
tail -2 $OUT/plain.log; for tool in memcheck initcheck synccheck racecheck; do echo "== $tool"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|rc=|SANITIZE_CASES_OK|Error" $OUT/sanitize_$tool.log | head -8; done

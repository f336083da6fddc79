#!/bin/bash
# compute-sanitizer over small launches of every library kernel (scripts/sanitize_workload.py):
# memcheck, racecheck (shared-memory hazards between the lanes/warps of a problem), synccheck and initcheck.
# Usage: sanitize.sh [TOOL...]   (default: all four).  Logs and a one-line verdict per tool in gpurun_out/sanitize/.
o=gpurun_out/sanitize; mkdir -p $o
python scripts/sanitize_workload.py > $o/plain.log 2>&1 || { echo "plain run failed"; tail -5 $o/plain.log; exit 1; }
tail -1 $o/plain.log
for tool in ${@:-memcheck racecheck synccheck initcheck}; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  [ $tool = initcheck ] && extra="--track-unused-memory no"
  timeout 3000 compute-sanitizer --tool $tool $extra --print-limit 30 --log-file $o/$tool.log \
    python scripts/sanitize_workload.py > $o/$tool.out 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $o/$tool.log | tail -1) : $(tail -1 $o/$tool.out)"
done

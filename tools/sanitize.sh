#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_cases.py) with
# memcheck, racecheck, synccheck and initcheck; one log per (tool, case) under
# gpurun_out/sanitize/, a summary line per run in gpurun_out/sanitize/summary.txt.
# Usage (on the GPU box): bash tools/sanitize.sh [case ...]
set -u
cd "$(dirname "$0")/.."
OUT=gpurun_out/sanitize
mkdir -p $OUT
CASES=${*:-sweep_band sweep_pruned_chunked band_overflow_exact sweep_groups train surrogate conv stereo raycast predict_merge records}
: > $OUT/summary.txt
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    extra=""
    [ $tool = memcheck ] && extra="--leak-check full"
    [ $tool = racecheck ] && extra="--racecheck-report all"
    log=$OUT/${tool}_${c}.txt
    timeout 900 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    errs=$(grep -Eo "ERROR SUMMARY: [0-9]+ error|RACECHECK SUMMARY: [0-9]+ hazard[s]? displayed \([0-9]+ error" $log | tail -1)
    ok=$(grep -c '"ok": true' $log)
    echo "$tool $c rc=$rc case_ok=$ok $errs" | tee -a $OUT/summary.txt
  done
done

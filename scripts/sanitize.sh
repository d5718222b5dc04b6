#!/bin/bash
# compute-sanitizer over scripts/sanitize_run.py (every kernel family on tiny
# shapes). Writes gpurun_out/sanitize_<tool>.log and a one-line summary per
# tool to gpurun_out/sanitize_summary.txt. NOTE: the graft GPU pool refuses
# compute-sanitizer (status 86, profiles/r02_sanitizer_refused.txt); this
# script is for machines where it is allowed.
#   bash scripts/sanitize.sh [racecheck synccheck memcheck initcheck]
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
tools=${*:-memcheck racecheck synccheck initcheck}
for t in $tools; do
  extra=""
  [ "$t" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool "$t" $extra --target-processes all --print-limit 50 \
      python scripts/sanitize_run.py > "gpurun_out/sanitize_$t.log" 2>&1
  rc=$?
  errs=$(grep -Eo "ERROR SUMMARY: [0-9]+ error" "gpurun_out/sanitize_$t.log" | tail -1)
  hz=$(grep -Eo "RACECHECK SUMMARY: [0-9]+ hazard[s]? displayed \([0-9]+ error[s]?, [0-9]+ warning[s]?\)" \
       "gpurun_out/sanitize_$t.log" | tail -1)
  ok=$(grep -c "sanitize ok" "gpurun_out/sanitize_$t.log")
  echo "$t rc=$rc ok=$ok ${errs} ${hz}" | tee -a gpurun_out/sanitize_summary.txt
done

#!/usr/bin/env bash
# compute-sanitizer over every kernel family at small n:
#   gpurun --timeout 3000 -- 'bash tools/sanitize.sh TAG'
# Logs: gpurun_out/TAG/sanitize_<tool>_<case>.log ; summary in status.txt.
set -u
TAG=${1:-r02_sanitize}
CASES=${2:-partition,quicksort,bps_stable,dist}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
python -c 'import paper_2004_12532_b200 as pp; pp.load()' > "$OUT/load.log" 2>&1
for tool in memcheck racecheck synccheck initcheck; do
  for c in ${CASES//,/ }; do
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 99 --print-limit 50 \
      python tests/sanitize_run.py --only $c > "$OUT/sanitize_${tool}_${c}.log" 2>&1
    rc=$?
    echo "$tool $c exit $rc" >> "$OUT/status.txt"
    grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" "$OUT/sanitize_${tool}_${c}.log" | tail -3 >> "$OUT/status.txt"
  done
done
cat "$OUT/status.txt"

#!/usr/bin/env bash
# compute-sanitizer over tools/sweep_cases.py (every kernel variant, small
# shapes): memcheck, racecheck (shared-memory hazards), synccheck (barrier
# misuse).  Logs land in gpurun_out/sanitizer_<tool>.log; summary lines on
# stdout.  CUDA graphs are disabled so every launch is seen individually.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=${CS:-/usr/local/cuda/bin/compute-sanitizer}
export PIDB_GRAPHS=0
for tool in memcheck synccheck racecheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report hazard"
  q=""
  [ "$tool" != memcheck ] && q="--quick"
  timeout 1500 "$CS" --tool "$tool" $extra --print-limit 50 --error-exitcode 99 \
      python tools/sweep_cases.py $q > "gpurun_out/sanitizer_${tool}.log" 2>&1
  echo "$tool rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitizer_${tool}.log | tail -1)"
done

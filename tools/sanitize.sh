#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py, one tool per run (run on the GPU box):
#   bash tools/sanitize.sh [outdir]   -> <outdir>/sanitize_<tool>.log
out=${1:-gpurun_out}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --error-exitcode 9 --print-limit 50 \
      python tools/sanitize_cases.py > "$out/sanitize_$tool.log" 2>&1
  echo "$tool rc=$?" | tee -a "$out/sanitize_summary.txt"
  tail -3 "$out/sanitize_$tool.log" >> "$out/sanitize_summary.txt"
done

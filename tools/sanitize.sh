#!/bin/bash
# Runs every case of tools/sanitize_cases.py under compute-sanitizer's memcheck,
# racecheck, synccheck and initcheck; one log per (tool, case) plus a summary.
#   bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out/sanitize}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
CASES="lat general graph_tma graph_reg batch sharded sparse analysis checkpoint"
: > "$OUT/summary.txt"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    log="$OUT/${tool}_${c}.log"
    timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 50 \
        python tools/sanitize_cases.py --case $c > "$log" 2>&1
    rc=$?
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$log" | tail -1)
    echo "$tool $c rc=$rc $errs" | tee -a "$OUT/summary.txt"
  done
done

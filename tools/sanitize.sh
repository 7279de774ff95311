#!/bin/bash
# compute-sanitizer over the sanitize subset (tests/test_sanitize.py), one pass per tool.
# Usage (on a GPU box): bash tools/sanitize.sh [outdir]   -> <outdir>/sanitize_<tool>.log
OUT=${1:-gpurun_out}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 1500 $CS --tool $tool $extra --target-processes all \
      --error-exitcode 99 --print-limit 50 \
      python -m pytest tests/test_sanitize.py -m sanitize -q -p no:cacheprovider > "$OUT/sanitize_$tool.log" 2>&1
  echo "$tool exit=$?" | tee -a "$OUT/sanitize_summary.txt"
  grep -E "ERROR SUMMARY|passed|failed" "$OUT/sanitize_$tool.log" | tail -3 | tee -a "$OUT/sanitize_summary.txt"
done

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over tools/sanitize_fits.py (summaries -> gpurun_out)
O=gpurun_out
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck initcheck; do
  arg=quick; [ $tool = memcheck ] && arg=full
  extra=""; [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 --error-exitcode 9 python tools/sanitize_fits.py $arg \
     > $O/san_$tool.log 2>&1
  echo "$tool rc=$?" | tee -a $O/san_summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Invalid|Race|Barrier|hazard" $O/san_$tool.log | head -20 >> $O/san_summary.txt
done

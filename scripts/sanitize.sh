#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_run.py
# (the cluster backward pass with its DSMEM slots and cluster barriers, the
# cooperative pass, cascade cancellation, seg2 cache, overlay). Logs under
# gpurun_out/; the summaries are copied into profiles/ by hand.
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 17 \
    python scripts/sanitize_run.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit $?" | tee -a gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log | tee -a gpurun_out/sanitize_summary.txt
done

#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck of the fused kernel
cd "$(dirname "$0")/.."
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 compute-sanitizer --tool $tool $extra --kernel-name regex:ndgi_fused --print-limit 50 \
     python scripts/sanitize.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done

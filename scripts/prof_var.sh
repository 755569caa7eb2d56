#!/bin/bash
# usage: scripts/prof_var.sh <name> [env assignments...]
cd "$(dirname "$0")/.."
NAME=$1; shift
for kv in "$@"; do export "$kv"; done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-vt"
timeout 300 $CMD > gpurun_out/${NAME}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 -o gpurun_out/${NAME} $CMD > gpurun_out/${NAME}_ncu.log 2>&1
echo done

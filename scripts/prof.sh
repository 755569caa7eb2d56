#!/bin/bash
# usage: scripts/prof.sh <name>  -- plain run then one ncu --set full capture of the fused kernel
cd "$(dirname "$0")/.."
NAME=${1:-prof}
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-vt > gpurun_out/${NAME}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 \
   -o gpurun_out/${NAME} python bench.py --steps 3 --warmup 3 --no-cpu --no-vt > gpurun_out/${NAME}_ncu.log 2>&1
echo done

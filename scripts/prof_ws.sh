#!/bin/bash
cd "$(dirname "$0")/.."
export NDGI_KERNEL=ws
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-vt"
timeout 300 $CMD > gpurun_out/pws_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 -o gpurun_out/prof_ws $CMD > gpurun_out/pws_ncu.log 2>&1
echo done

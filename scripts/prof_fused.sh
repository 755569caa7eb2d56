#!/bin/bash
# ncu --set full capture (with source) of the bench's fused-kernel launch, plus
# the per-SASS-instruction CSV; usage: scripts/prof_fused.sh TAG [extra bench args]
cd "$(dirname "$0")/.."
TAG=${1:-prof}; shift
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit $*"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 \
   -o gpurun_out/${TAG}_fused $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
if [ -f gpurun_out/${TAG}_fused.ncu-rep ]; then
  python scripts/ncu_summary.py gpurun_out/${TAG}_fused.ncu-rep > gpurun_out/${TAG}_fused.txt 2>&1
  ncu -i gpurun_out/${TAG}_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
  gzip -f gpurun_out/${TAG}_src.csv
  find gpurun_out -name '*.ncu-rep' -size +40M -delete
fi

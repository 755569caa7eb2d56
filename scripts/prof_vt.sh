#!/bin/bash
# ncu --set full (with source) of one VT batch kernel (config 3, n = $2)
cd "$(dirname "$0")/.."
TAG=${1:-vt}; N=${2:-8}
timeout 300 python scripts/vt_probe.py $N > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 5 -c 1 \
   -o gpurun_out/${TAG} python scripts/vt_probe.py $N > gpurun_out/${TAG}_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/${TAG}.ncu-rep > gpurun_out/${TAG}.txt 2>&1
ncu -i gpurun_out/${TAG}.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
gzip -f gpurun_out/${TAG}_src.csv
find gpurun_out -name '*.ncu-rep' -size +40M -delete

#!/bin/bash
cd "$(dirname "$0")/.."
T=${1:-aux}
python scripts/aux_probe.py train > gpurun_out/${T}_train_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_train_grad -s 3 -c 1 -o gpurun_out/${T}_train python scripts/aux_probe.py train > gpurun_out/${T}_train_ncu.log 2>&1
python scripts/aux_probe.py sample > gpurun_out/${T}_sample_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_sample -s 3 -c 1 -o gpurun_out/${T}_sample python scripts/aux_probe.py sample > gpurun_out/${T}_sample_ncu.log 2>&1
for k in train sample; do
  python scripts/ncu_summary.py gpurun_out/${T}_$k.ncu-rep > gpurun_out/${T}_$k.txt 2>&1
  ncu -i gpurun_out/${T}_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/${T}_${k}_src.csv 2>/dev/null; gzip -f gpurun_out/${T}_${k}_src.csv
done
find gpurun_out -name '*.ncu-rep' -size +40M -delete
cat gpurun_out/${T}_train_plain.log gpurun_out/${T}_sample_plain.log

#!/bin/bash
# finer tail units vs whole-tile tail: residency probe + same-box bench A/B + the new parity test
cd "$(dirname "$0")/.."
python scripts/residency_probe.py c2 > gpurun_out/res3.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -k "dynamic_schedule or c2_bench or batch_equals" > gpurun_out/tests3.log 2>&1; echo "rc=$?" >> gpurun_out/tests3.log
bash scripts/variants.sh abt base notail > gpurun_out/ab_tail.txt 2>&1
for cell in c5:H:bc7 c5:M64:bc7 c5:L:bc7; do
  for v in base notail; do
    if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
    echo "$cell $v $(python scripts/cell_time.py $cell 2>&1 | tail -1)" >> gpurun_out/ab_tail.txt
  done
done

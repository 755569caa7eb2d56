#!/bin/bash
# dynamic vs static unit scheduling: residency probe + same-box bench A/B + decode tests
cd "$(dirname "$0")/.."
python scripts/residency_probe.py c2 > gpurun_out/res2.txt 2>&1
python scripts/residency_probe.py c5:H:bc7 >> gpurun_out/res2.txt 2>&1
bash scripts/variants.sh ab base static > gpurun_out/ab_sched.txt 2>&1
for cell in c5:H:bc7 c5:M64:bc7; do
  for v in base static; do
    if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
    echo "$cell $v $(python scripts/cell_time.py $cell 2>&1 | tail -1)" >> gpurun_out/ab_sched.txt
  done
done
unset NDGI_LIB
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests2.log 2>&1; echo "rc=$?" >> gpurun_out/tests2.log

#!/bin/bash
# MUFU/FMA GELU split re-swept under dynamic scheduling + ncu of the bench launch
cd "$(dirname "$0")/.."
bash scripts/variants.sh abp base p22 p32 p33 p11 > gpurun_out/ab_poly.txt 2>&1
for cell in c5:H:bc7; do
  for v in base p22 p32; do
    if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
    echo "$cell $v $(python scripts/cell_time.py $cell 2>&1 | tail -1)" >> gpurun_out/ab_poly.txt
  done
done
unset NDGI_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 -o gpurun_out/r2b_M python bench.py --steps 3 --warmup 3 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/r2b_M_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2b_M.ncu-rep > gpurun_out/r2b_M.txt 2>&1

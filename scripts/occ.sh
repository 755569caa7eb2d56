#!/bin/bash
cd "$(dirname "$0")/.."
for v in "" occ7 occ8; do
  if [ -n "$v" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  NDGI_VERBOSE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-vt > gpurun_out/occ_$v.log 2>&1
done
echo done

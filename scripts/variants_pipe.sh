#!/bin/bash
cd "$(dirname "$0")/.."
for v in "$@"; do
  export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so
  NDGI_KERNEL=pipe timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/var_$v.log 2>&1
done
echo done

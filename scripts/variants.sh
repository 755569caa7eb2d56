#!/bin/bash
# usage: scripts/variants.sh v1 v2 ... -- bench each libndgi_<v>.so ("" = default build)
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/var_$v.log 2>&1
done
echo done

#!/bin/bash
# h = 64 GELU split: M.64 cell time per variant (base = 1 poly pair of 8)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for v in base m64p2 m64p3; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  echo "M64 $v $(python scripts/cell_time.py c5:M64:bc7 2>&1 | tail -1)"
done
done

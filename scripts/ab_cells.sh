#!/bin/bash
# A/B of config-5 cells: scripts/ab_cells.sh TAG cell1,cell2 v1 v2 ... (v = base | variant lib name)
cd "$(dirname "$0")/.."
TAG=$1; CELLS=$2; shift 2
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  python scripts/cell_time.py $CELLS | sed "s/^/$v $rep /"
done
done

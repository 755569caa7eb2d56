#!/bin/bash
# usage: scripts/ab_run.sh TAG v1 v2 ... : c2 bench A/B (variants.sh) + H cell times per variant
cd "$(dirname "$0")/.."
TAG=$1; shift
bash scripts/variants.sh $TAG "$@" > gpurun_out/$TAG.txt 2>&1
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  echo "H $v $(python scripts/cell_time.py c5:H:bc7 2>&1 | tail -1)" >> gpurun_out/$TAG.txt
done
cat gpurun_out/$TAG.txt

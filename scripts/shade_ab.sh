#!/bin/bash
# A/B of the shading leg: scripts/shade_ab.sh v1 v2 ...
cd "$(dirname "$0")/.."
for rep in 1 2; do for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  python -c "
import sys; sys.argv=['bench.py']; import bench, torch, paper_2604_12625_b200 as ndgi, argparse
r=bench.shading_leg(ndgi, torch, argparse.Namespace()); print('$v', $rep, round(r['sample_kernel_us'],2), round(r['roofline']['frac'],3))"
done; done

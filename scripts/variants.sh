#!/bin/bash
# usage: scripts/variants.sh TAG v1 v2 ... -- times the c2 bench step for each
# libndgi_<v>.so ("base" = the default build), twice, interleaved
cd "$(dirname "$0")/.."
TAG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit \
     > gpurun_out/${TAG}_${v}_$rep.json 2> gpurun_out/${TAG}_${v}_$rep.err
  python -c "import json,sys; d=json.loads(open('gpurun_out/${TAG}_${v}_$rep.json').read().splitlines()[-1]); print('$v', '$rep', round(d['value'],2), round(d['roofline']['frac'],3))" 2>/dev/null || echo "$v $rep FAILED"
done
done

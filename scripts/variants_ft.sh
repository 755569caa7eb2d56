#!/bin/bash
# usage: scripts/variants_ft.sh v1 v2 ... -- fine-tune / full-step legs of each libndgi_<v>.so ("base" = default build)
cd "$(dirname "$0")/.."
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-vt --no-shading --no-texunit --no-encode > gpurun_out/ft_$v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ft_$v.log').read().strip().splitlines()[-1]); print('$v', d['finetune']['ms_per_step'], d['finetune']['full']['ms_per_step'])"
done

#!/bin/bash
# A/B of the VT leg: scripts/vt_ab.sh TAG v1 v2 ...
cd "$(dirname "$0")/.."
TAG=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/${TAG}_${v}_$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/${TAG}_${v}_$rep.json').read().splitlines()[-1]); v=d['vt_batch_us']; print('$v', $rep, {k: (round(x['p50'],1), round(x.get('device_p50',0),1)) for k,x in v.items() if isinstance(x, dict)})"
done; done

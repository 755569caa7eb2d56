#!/bin/bash
# usage: scripts/variants_t.sh v1 v2 ... -- quick parity test + bench of each libndgi_<v>.so
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
for v in "$@"; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "fast_full_parity or tiles_border or strips" 2>&1 | tail -1 > gpurun_out/vt_$v.log
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/var_$v.log 2>&1
done
echo done

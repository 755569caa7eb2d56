#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
export NDGI_KERNEL=hmma
timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "fast or cross or batch or strips or bad or host or c2" 2>&1 | tail -15 > gpurun_out/hm_tests.log
for v in base hm6 hm5 hm4; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/hm_$v.log 2>&1
done
echo done

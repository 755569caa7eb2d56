#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
NDGI_KERNEL=ws timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "fast or cross or batch or strips or bad or host or c2" 2>&1 | tail -15 > gpurun_out/ws_tests.log
NDGI_KERNEL=ws NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/ws_bench.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/v6_bench.log 2>&1
echo done

#!/bin/bash
# tests + bench of the CTA-synchronous h=16 kernel (NDGI_KERNEL=sync) and of the default
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
NDGI_KERNEL=sync timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -5 > gpurun_out/sync_tests.log
NDGI_KERNEL=sync NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/sync_bench.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/pipe_bench.log 2>&1
echo done

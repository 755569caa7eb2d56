#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -15 > gpurun_out/pipe_tests.log
NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/pipe_bench.log 2>&1
NDGI_KERNEL=sync timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/sync_bench.log 2>&1
echo done

#!/bin/bash
# parity tests + bench of the pipelined h=16 kernel (NDGI_KERNEL=pipe)
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
NDGI_KERNEL=pipe timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -5 > gpurun_out/pipe_tests.log
NDGI_KERNEL=pipe NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/pipe_bench.log 2>&1
echo done

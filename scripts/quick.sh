#!/bin/bash
# GPU parity tests + a short bench of the default build (usage: scripts/quick.sh [tag])
cd "$(dirname "$0")/.."
T=${1:-q}
python -c "import oracle; oracle.build()"
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q 2>&1 | tail -5 > gpurun_out/${T}_tests.log
NDGI_VERBOSE=1 timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu --no-vt > gpurun_out/${T}_bench.log 2>&1
echo done

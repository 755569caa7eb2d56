#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15 > gpurun_out/t_all.log
NDGI_VERBOSE=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-vt > gpurun_out/b_small.log 2>&1
bash scripts/prof.sh prof_v6
echo done

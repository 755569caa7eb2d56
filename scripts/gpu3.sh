#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5 > gpurun_out/t_all.log
NDGI_VERBOSE=1 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-vt > gpurun_out/b_small.log 2>&1
timeout 600 python bench.py --no-cpu > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 \
   -o gpurun_out/prof_fused python bench.py --steps 3 --warmup 3 --no-cpu --no-vt > gpurun_out/ncu_full.log 2>&1
echo done

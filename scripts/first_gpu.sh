#!/bin/bash
# first GPU trip: build check, BC7 + ref + fast parity, gelu rate
cd "$(dirname "$0")/.."
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import oracle; oracle.build()"
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -s -k "bc7" 2>&1 | tail -20 > gpurun_out/t_bc7.log
timeout 600 python -m pytest tests/test_gpu_decode.py -x -q -s -k "ref_fp32" 2>&1 | tail -30 > gpurun_out/t_ref.log
timeout 300 python -c "
import paper_2604_12625_b200 as n
ms, a = n.ndgi_debug_gelu_rate(2048)
print('gelu rate', a/ms/1e6, 'G act/s', ms, 'ms')
" > gpurun_out/gelu.log 2>&1
timeout 300 python -m pytest tests/test_gpu_decode.py -q -s -k "fast or cross or batch or strips or bad or host" 2>&1 | tail -60 > gpurun_out/t_fast.log
echo done

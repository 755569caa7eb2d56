#!/bin/bash
cd "$(dirname "$0")/.."
python -c "import oracle; oracle.build()"
for k in "texture_unit_agrees or tiles_border" "parity and H or tiles_border" "parity and C256 or tiles_border" "parity and M64 or tiles_border" "bc7_device or tiles_border" "ref_fp32 or tiles_border"; do
  echo "== $k"; timeout 300 python -m pytest tests/test_gpu_decode.py -x -q -k "$k" 2>&1 | tail -2
done

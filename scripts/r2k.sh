timeout 1500 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_regimes.py tests/test_gpu_selfcheck.py -q -x -p no:cacheprovider > gpurun_out/r2k_tests.log 2>&1
tail -2 gpurun_out/r2k_tests.log
bash scripts/ab_cells.sh r2k c2,c5:H:bc7,c5:H:u8,c5:H:bc3 base old

set -x
timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_regimes.py -q -x -p no:cacheprovider > gpurun_out/r2c_tests.log 2>&1
tail -3 gpurun_out/r2c_tests.log
bash scripts/variants.sh r2c base spinhint p11 p22 p32 p00

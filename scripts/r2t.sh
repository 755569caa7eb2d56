timeout 1200 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_regimes.py tests/test_gpu_selfcheck.py -q -x -p no:cacheprovider > gpurun_out/r2t_tests.log 2>&1; tail -2 gpurun_out/r2t_tests.log
python scripts/vt_timeline.py
bash scripts/vt_ab.sh r2t base old

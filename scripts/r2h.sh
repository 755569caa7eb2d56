timeout 1200 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_regimes.py tests/test_gpu_train.py tests/test_gpu_train_full.py -q -x -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1
tail -2 gpurun_out/r2h_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/r2h.json 2> gpurun_out/r2h.err
python -c "import json; d=json.loads(open('gpurun_out/r2h.json').read().splitlines()[-1]); print(d['value'], d['roofline']['frac']); v=d['vt_batch_us']; print({k: (round(x['p50'],1), round(x.get('device_p50',0),1)) for k,x in v.items() if isinstance(x, dict)})"
python scripts/sweep.py > gpurun_out/r2h_sweep.json 2> gpurun_out/r2h_sweep.err; tail -3 gpurun_out/r2h_sweep.json

timeout 900 python -m pytest tests/test_gpu_decode.py tests/test_gpu_parity_regimes.py -q -x -p no:cacheprovider > gpurun_out/r2e_tests.log 2>&1
tail -2 gpurun_out/r2e_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/r2e_vt.json 2> gpurun_out/r2e_vt.err
python -c "import json; d=json.loads(open('gpurun_out/r2e_vt.json').read().splitlines()[-1]); print(d['value'], d['roofline']['frac']); print(json.dumps(d['vt_batch_us']))"
bash scripts/host_overhead.sh > gpurun_out/r2e_host.log 2>&1; cat gpurun_out/r2e_host.log

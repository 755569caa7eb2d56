timeout 900 python -m pytest tests/test_gpu_decode.py -q -x -p no:cacheprovider -k "strip or tiles or small or windowed or bench_launch" > gpurun_out/r2f_tests.log 2>&1
tail -2 gpurun_out/r2f_tests.log
for v in base nopf; do
  if [ "$v" != "base" ]; then export NDGI_LIB=$PWD/paper_2604_12625_b200/libndgi_$v.so; else unset NDGI_LIB; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/r2f_$v.json 2> gpurun_out/r2f_$v.err
  python -c "import json; d=json.loads(open('gpurun_out/r2f_$v.json').read().splitlines()[-1]); print('$v', d['value'], d['roofline']['frac']); v=d['vt_batch_us']; print({k: (round(x['p50'],1), round(x.get('device_p50',0),1)) for k,x in v.items() if isinstance(x, dict)})"
done

bash scripts/variants.sh r2d base tid0 onepoll cwait tid0cw tid0op
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/r2d_vt.json 2> gpurun_out/r2d_vt.err
python -c "import json; d=json.loads(open('gpurun_out/r2d_vt.json').read().splitlines()[-1]); print(json.dumps(d['vt_batch_us']))"

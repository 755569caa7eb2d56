timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1
tail -4 gpurun_out/r2m_tests.log
timeout 900 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r2m_bench.json').read().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['roofline']['peak'], d['e2e']['value'])"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2m_ref.json 2> gpurun_out/r2m_ref.err; tail -c 300 gpurun_out/r2m_ref.json

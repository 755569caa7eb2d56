#!/bin/bash
# round-2 capture: GPU tests, default bench line, c4 path, config-5 sweep, ncu
cd "$(dirname "$0")/.."
T=${1:-r2f}
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${T}_tests.log 2>&1; tail -3 gpurun_out/${T}_tests.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; tail -c 200 gpurun_out/${T}_bench.json
timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/${T}_c4.json 2> gpurun_out/${T}_c4.err; tail -c 200 gpurun_out/${T}_c4.json
timeout 1200 python scripts/sweep.py > gpurun_out/${T}_sweep.json 2> gpurun_out/${T}_sweep.err; tail -c 200 gpurun_out/${T}_sweep.json
bash scripts/round_capture.sh ${T}
python scripts/residency_probe.py c2 > gpurun_out/${T}_residency.txt 2>&1
RES_LIB=libndgi_res.so python scripts/residency_probe.py c5:H:bc7 >> gpurun_out/${T}_residency.txt 2>&1
python scripts/ncu_summary.py gpurun_out/${T}_M.ncu-rep gpurun_out/${T}_launches.csv > gpurun_out/${T}_M.txt 2>&1

#!/bin/bash
# Round capture: GPU tests, default bench line, ncu launch list of the bench, one
# ncu --set full capture of the fused kernel.  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
TAG=${1:-r1}
python -c "import oracle; oracle.build()"
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -5 > gpurun_out/${TAG}_tests.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --no-vt"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 \
   -o gpurun_out/${TAG}_fused $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1

# summaries on the box (the full report can exceed gpurun's 64 MiB copy-back)
if [ -f gpurun_out/${TAG}_fused.ncu-rep ]; then
  python scripts/ncu_summary.py gpurun_out/${TAG}_fused.ncu-rep gpurun_out/${TAG}_launches.csv > gpurun_out/${TAG}_fused.txt 2>&1
  python scripts/ncu_hot.py gpurun_out/${TAG}_fused.ncu-rep 40 > gpurun_out/${TAG}_fused_hot_sass.txt 2>&1
  ncu -i gpurun_out/${TAG}_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
  python scripts/ncu_regions.py gpurun_out/${TAG}_src.csv > gpurun_out/${TAG}_fused_regions.txt 2>&1
  rm -f gpurun_out/${TAG}_src.csv
  find gpurun_out -name '*.ncu-rep' -size +40M -delete
fi
echo done

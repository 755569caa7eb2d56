#!/bin/bash
# Round capture: ncu launch list of the default bench command, and one
# `ncu --set full` capture (with source) of the fused kernel for config 2 (M,
# the bench launch), the H profile and M.64 (config 5 cells).  Outputs in gpurun_out/.
cd "$(dirname "$0")/.."
TAG=${1:-r2}
CMD="python bench.py --steps 3 --warmup 3"
timeout 900 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
cap() {   # cap NAME CMD...
  local name=$1; shift
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 \
     -o gpurun_out/${TAG}_$name "$@" > gpurun_out/${TAG}_${name}_ncu.log 2>&1
  python scripts/ncu_summary.py gpurun_out/${TAG}_$name.ncu-rep > gpurun_out/${TAG}_$name.txt 2>&1
  ncu -i gpurun_out/${TAG}_$name.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_${name}_src.csv 2>/dev/null
  gzip -f gpurun_out/${TAG}_${name}_src.csv
}
cap M python bench.py --steps 3 --warmup 3 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit
cap H python scripts/c5_probe.py c5:H:bc7
cap M64 python scripts/c5_probe.py c5:M64:bc7
# gpurun copies back at most 64 MiB: keep the bench kernel's report, the
# others as their text summaries and source pages
rm -f gpurun_out/${TAG}_H.ncu-rep gpurun_out/${TAG}_M64.ncu-rep
echo done

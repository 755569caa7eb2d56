timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 -o gpurun_out/r2o_H python scripts/c5_probe.py c5:H:bc7 > gpurun_out/r2o_H_ncu.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2o_H.ncu-rep > gpurun_out/r2o_H.txt 2>&1
ncu -i gpurun_out/r2o_H.ncu-rep --page source --csv --print-source sass > gpurun_out/r2o_H_src.csv 2>/dev/null; gzip -f gpurun_out/r2o_H_src.csv

cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c1_smi.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/c1_gputests.log 2>&1
echo "tests rc=$?" >> gpurun_out/c1_gputests.log
timeout 600 python bench.py > gpurun_out/c1_bench.json 2> gpurun_out/c1_bench.err
echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ndgi_fused -s 3 -c 1 -o gpurun_out/c1_M python bench.py --steps 3 --warmup 3 --no-cpu --no-vt --no-shading --no-encode --no-finetune --no-texunit > gpurun_out/c1_M_ncu.log 2>&1
ncu -i gpurun_out/c1_M.ncu-rep --page raw --csv > gpurun_out/c1_M_raw.csv 2>&1
echo done

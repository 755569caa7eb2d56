cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "H or ring or RING or R3 or bc1 or bc3 or windowed or c5 or selfcheck or tiles or strip" > gpurun_out/q2_tests.log 2>&1; tail -3 gpurun_out/q2_tests.log
bash scripts/ab_cells.sh q2 c5:H:bc7,c5:H:u8,c5:H:f16,c5:M:bc7,c5:L:bc7 base stage

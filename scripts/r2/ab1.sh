export PYTEST_TARGETS="tests/test_gpu_parity.py"
export PYTEST_K="strip_spread or config1 or smooth_part_vs_direct or config2_full"
export VARIANTS="pair
old --opt spread_pack=2"
bash scripts/r2/gpu_ab.sh
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_interp_local|k_tri_local|k_local_stencil" -c 4 -o gpurun_out/prof/full_pair python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_pair.log 2>&1; echo ncu=$?

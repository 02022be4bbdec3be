# A/B + profile: four-step columns with cp.async loads; ncu of the pair spreader and the interp/local kernels
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab2.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or smooth_gate_full_c4 or strip" > gpurun_out/pytest_ab2.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab2_pair.json 2> gpurun_out/ab2_pair.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_fft4|k_interp_local|k_tri_local|k_local_stencil" -c 8 -o gpurun_out/prof/full_ab2 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab2.log 2>&1; echo ncu=$?

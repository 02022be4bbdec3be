# pair spreader with precomputed offsets, chunk prefetch; interp with paired Horner taps
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab3.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "strip or config1 or config2_full or smooth_part or off_node" > gpurun_out/pytest_ab3.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab3.json 2> gpurun_out/ab3.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_interp_local" -c 2 -o gpurun_out/prof/full_ab3 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab3.log 2>&1; echo ncu=$?

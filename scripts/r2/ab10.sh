# fused prolongation with compile-time taps; cp.async in the restriction; k_fft4_b row tables
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab10.json timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or config1 or config5 or smooth_gate" > gpurun_out/pytest_ab10.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab10.json 2> gpurun_out/ab10.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row4_inv|k_restrict|k_fft4_b" -c 5 -o gpurun_out/prof/full_ab10 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab10.log 2>&1; echo ncu=$?

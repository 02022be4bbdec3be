# cluster-pair row passes; fused TRIANGLE tail (interp -> vH, k_tri_out -> out)
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab6.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or strip or config1 or config4 or batch" > gpurun_out/pytest_ab6.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab6.json 2> gpurun_out/ab6.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt fft_rows=1 > gpurun_out/ab6_rows.json 2> gpurun_out/ab6_rows.err; echo bench=$?
VP_OPTS="fft_rows=1" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row4|k_tri_out|k_interp_local" -c 6 -o gpurun_out/prof/full_ab6 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab6.log 2>&1; echo ncu=$?

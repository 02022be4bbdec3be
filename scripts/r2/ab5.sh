# full-row own row passes (both half-sequences per CTA)
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab5.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step" > gpurun_out/pytest_ab5.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt fft_rows=1 > gpurun_out/ab5_rows.json 2> gpurun_out/ab5_rows.err; echo bench=$?
VP_OPTS="fft_rows=1" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row4" -c 4 -o gpurun_out/prof/full_ab5rows python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab5rows.log 2>&1; echo ncu=$?

# full-row own row passes at 1024 threads; pair spreader with the odd-row predicate
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab7.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or strip or config1" > gpurun_out/pytest_ab7.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt fft_rows=1 > gpurun_out/ab7_rows.json 2> gpurun_out/ab7_rows.err; echo bench=$?
VP_OPTS="fft_rows=1" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row4|k_spread_pair" -c 5 -o gpurun_out/prof/full_ab7 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab7.log 2>&1; echo ncu=$?

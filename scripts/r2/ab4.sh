# two accumulator rings in the pair spreader; own row passes profiled
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab4.json timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "strip or config1 or four_step" > gpurun_out/pytest_ab4.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab4.json 2> gpurun_out/ab4.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt fft_rows=1 > gpurun_out/ab4_rows.json 2> gpurun_out/ab4_rows.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair" -c 1 -o gpurun_out/prof/full_ab4 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab4.log 2>&1; echo ncu=$?
VP_OPTS="fft_rows=1" timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_row4" -c 2 -o gpurun_out/prof/full_ab4rows python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab4rows.log 2>&1; echo ncu=$?

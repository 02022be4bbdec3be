# fused prolongation in the NH inverse rows; pair strips 128 rows tall
set -x
mkdir -p gpurun_out/prof
VP_PARITY_LOG=gpurun_out/parity_ab9.json timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or strip or config1 or config4 or config5 or batch" > gpurun_out/pytest_ab9.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab9.json 2> gpurun_out/ab9.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_row4_inv" -c 3 -o gpurun_out/prof/full_ab9 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab9.log 2>&1; echo ncu=$?

set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "eval_batch" > gpurun_out/pytest_b3.log 2>&1; echo pytest=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_spread_strip_b" -s 1 -c 1 python scripts/one_eval_batch.py c5 4 > gpurun_out/ncu_batch_c5.log 2>&1; echo n=$?

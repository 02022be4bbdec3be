set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "strip or config2 or config5 or eval_batch or determin or tiny" > gpurun_out/pytest_s8.log 2>&1; echo pytest=$?
timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5.json 2>&1; echo p5=$?
timeout 600 python scripts/probe_spread.py c2 > gpurun_out/probe_spread_c2.json 2>&1; echo p2=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_spread_strip|k_scatter_f" -s 2 -c 2 python scripts/one_eval.py c5 0 2 > gpurun_out/ncu_s8_c5.log 2>&1; echo n5=$?

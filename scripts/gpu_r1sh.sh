set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "strip or config2 or eval_batch" > gpurun_out/pytest_sh.log 2>&1; echo pytest=$?
timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5.json 2>&1; echo p5=$?
timeout 600 python scripts/probe_spread.py c2 > gpurun_out/probe_spread_c2.json 2>&1; echo p2=$?

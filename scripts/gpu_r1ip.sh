set -x
timeout 1500 python -m pytest tests -m gpu -q -x -k "config1 or config2 or config5 or off_node or tiny or determin or loose or batch" > gpurun_out/pytest_ip.log 2>&1; echo pytest=$?
timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5.json 2>&1; echo p5=$?
timeout 600 python scripts/probe_spread.py c2 > gpurun_out/probe_spread_c2.json 2>&1; echo p2=$?

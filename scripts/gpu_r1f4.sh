set -x
timeout 600 python scripts/probe_fft.py c2 > gpurun_out/probe_fft_c2.json 2>&1; echo p2=$?
timeout 600 python scripts/probe_fft.py c1 > gpurun_out/probe_fft_c1.json 2>&1; echo p1=$?
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_fft or config1 or config2 or smooth or loose or tiny" > gpurun_out/pytest_fft.log 2>&1; echo pytest=$?

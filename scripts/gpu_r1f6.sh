set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "fused_fft" > gpurun_out/pytest_fft.log 2>&1; echo pytest=$?
timeout 900 python scripts/probe_fft.py c4 > gpurun_out/probe_fft_c4.json 2>&1; echo p4=$?
timeout 1200 python scripts/probe_fft.py c5 > gpurun_out/probe_fft_c5.json 2>&1; echo p5=$?
timeout 900 python scripts/probe_fft.py c3 > gpurun_out/probe_fft_c3.json 2>&1; echo p3=$?

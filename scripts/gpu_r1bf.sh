set -x
timeout 600 python scripts/sanitize_small.py > gpurun_out/all_paths.log 2>&1; echo ap=$?
timeout 1200 python -m pytest tests -m gpu -q -x -k "config3 or fused_fft or config2 or smooth" > gpurun_out/pytest_bf.log 2>&1; echo pytest=$?
timeout 900 python scripts/probe_fft.py c3 > gpurun_out/probe_fft_c3.json 2>&1; echo p3=$?

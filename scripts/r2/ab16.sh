# single layer on the star (delta convergence) + the full GPU suite after adding vp_layer.cu
set -x
mkdir -p gpurun_out/ab16
timeout 1200 python -m pytest tests/test_layer.py -m gpu -q -s > gpurun_out/ab16/pytest_layer.log 2>&1; echo pytest=$?

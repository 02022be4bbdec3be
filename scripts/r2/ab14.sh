# single-layer potential: GPU parity
set -x
mkdir -p gpurun_out/ab14
timeout 1200 python -m pytest tests/test_layer.py -m gpu -q -s > gpurun_out/ab14/pytest.log 2>&1; echo pytest=$?

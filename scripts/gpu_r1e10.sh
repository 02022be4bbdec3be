set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "eval_batch" > gpurun_out/pytest_b4.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?

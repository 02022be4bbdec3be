set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "eval_batch" > gpurun_out/pytest_bc.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_bc.json 2> gpurun_out/bench_c2_bc.err; echo b2=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3_bc.json 2> gpurun_out/bench_c3_bc.err; echo b3=$?

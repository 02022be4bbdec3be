set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "eval_batch or strip or fused_fft" > gpurun_out/pytest_batch.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c2_b.json 2> gpurun_out/bench_c2_b.err; echo b2=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/bench_c5_b.json 2> gpurun_out/bench_c5_b.err; echo b5=$?

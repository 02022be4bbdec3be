set -x
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?

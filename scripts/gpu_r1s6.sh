set -x
timeout 1200 python -m pytest tests -m gpu -q -k "config3 or strip or tiny or determin" > gpurun_out/pytest_c3.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c3.csv python scripts/one_eval.py c3 0 1 > gpurun_out/ncu_launch_c3.log 2>&1; echo l3=$?

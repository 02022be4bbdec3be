set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s -k "not config3" > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
python bench.py --steps 2 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/plain5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/ncu_launch5.log 2>&1; echo ncu5=$?

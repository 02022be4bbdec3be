set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
python bench.py --steps 2 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/plain5.log 2>&1 && \
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:"k_interp_local|k_spread_nh" -s 2 -c 2 -o gpurun_out/prof_c5d python bench.py --steps 1 --warmup 2 --config c5 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo ncu5=$?

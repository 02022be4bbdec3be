set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ncu_launch_c2.log 2>&1; echo l2=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip|k_interp_local|k_local_stencil|k_fft" -s 6 -c 8 -o gpurun_out/prof_c2_e4 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ncu_c2.log 2>&1; echo ncu2=$?

set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c4 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref.err; echo ref=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l2.log 2>&1; echo ncul=$?

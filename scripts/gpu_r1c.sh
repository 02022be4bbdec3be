set -x
free -g; nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 600 python scripts/probe_c3.py small 512 256 > gpurun_out/probe_c3s.json 2>&1; echo c3s=$?
timeout 900 python scripts/probe_c3.py full 256 128 > gpurun_out/probe_c3.json 2>&1; echo c3=$?
timeout 1500 python scripts/probe_configs.py c5 > gpurun_out/probe_c5.json 2>&1; echo c5=$?
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_nh|k_interp_local|k_restrict_x" -s 3 -c 3 -o gpurun_out/prof_c2c python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

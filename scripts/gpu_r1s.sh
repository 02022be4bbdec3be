set -x
timeout 600 python bench.py --steps 2 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/plain5.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spread_dense|k_spread_nh" -s 2 -c 2 -o gpurun_out/prof_c5h python bench.py --steps 1 --warmup 2 --config c5 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo ncu5=$?

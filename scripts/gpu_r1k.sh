set -x
python bench.py --steps 2 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/plain5.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 1 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/ncu_launch5.log 2>&1; echo ncu5=$?
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_nh|k_interp_local|k_local_stencil|k_restrict|k_prolong" -s 6 -c 6 -o gpurun_out/prof_c2f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?

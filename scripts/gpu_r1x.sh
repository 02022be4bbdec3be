set -x
timeout 600 python bench.py --steps 2 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/plain3.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 1 --warmup 2 --config c3 --no-cpu-baseline > gpurun_out/ncu_l3.log 2>&1; echo ncul=$?

set -x
timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5.json 2>&1; echo p5=$?
VP_STRIP_SIZE_ORDER=1 timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5_size.json 2>&1; echo p5s=$?
timeout 600 python scripts/probe_spread.py c2 > gpurun_out/probe_spread_c2.json 2>&1; echo p2=$?
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum --clock-control none -k regex:"k_spread_strip" -s 1 -c 1 python scripts/one_eval.py c5 0 2 > gpurun_out/ncu_strip_c5_dram.log 2>&1; echo n5=$?

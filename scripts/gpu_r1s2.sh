set -x
timeout 600 python scripts/one_eval.py c5 0 2 > gpurun_out/one_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip" -s 1 -c 1 -o gpurun_out/prof_strip_c5 python scripts/one_eval.py c5 0 2 > gpurun_out/ncu_strip_c5.log 2>&1; echo n5=$?
timeout 600 python scripts/one_eval.py c2 0 2 > gpurun_out/one_c2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip" -s 1 -c 1 -o gpurun_out/prof_strip_c2 python scripts/one_eval.py c2 0 2 > gpurun_out/ncu_strip_c2.log 2>&1; echo n2=$?

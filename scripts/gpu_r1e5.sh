set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip|k_interp_local|k_tri_local12|k_local_stencil|k_fft" -s 5 -c 6 -o gpurun_out/prof_c4_e5 python scripts/one_eval.py c4 0 2 > gpurun_out/ncu_c4.log 2>&1; echo n4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip|k_interp_local|k_band_sum|k_fft" -s 8 -c 10 -o gpurun_out/prof_c3_e5 python scripts/one_eval.py c3 0 2 > gpurun_out/ncu_c3.log 2>&1; echo n3=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c5.csv python scripts/one_eval.py c5 0 2 > gpurun_out/ncu_launch_c5.log 2>&1; echo l5=$?

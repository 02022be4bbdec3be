timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|fft|process_kernel" -c 400 --csv --log-file /tmp/launches_c5.csv python scripts/one_eval.py c5 0 2 > /tmp/ncu_launch_c5.log 2>&1; echo l5=$?
gzip -c /tmp/launches_c5.csv > gpurun_out/launches_c5_r1final.csv.gz

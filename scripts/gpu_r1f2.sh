timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fft" -c 6 -o gpurun_out/prof_fft_c2 python scripts/one_eval.py c2 0 2 > gpurun_out/ncu_fft_c2.log 2>&1; echo n=$?

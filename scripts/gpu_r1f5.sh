set -x
timeout 900 python scripts/probe_fft.py c3 > gpurun_out/probe_fft_c3.json 2>&1; echo p3=$?
timeout 900 python scripts/probe_fft.py c4 > gpurun_out/probe_fft_c4.json 2>&1; echo p4=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_fft" -c 6 -o gpurun_out/prof_fft_c2b python scripts/one_eval.py c2 0 2 > gpurun_out/ncu_fft_c2.log 2>&1; echo n=$?

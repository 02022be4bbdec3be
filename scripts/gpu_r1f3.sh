set -x
timeout 600 python scripts/probe_fft.py c2 > gpurun_out/probe_fft_c2.json 2>&1; echo p2=$?
timeout 900 python scripts/probe_fft.py c3 > gpurun_out/probe_fft_c3.json 2>&1; echo p3=$?
timeout 900 python scripts/probe_fft.py c4 > gpurun_out/probe_fft_c4.json 2>&1; echo p4=$?

set -x
timeout 900 python scripts/probe_tiles.py c2 > gpurun_out/probe_tiles_c2.json 2>&1; echo t2=$?
timeout 1500 python scripts/probe_tiles.py c5 > gpurun_out/probe_tiles_c5.json 2>&1; echo t5=$?

for d in 0 1 2 3; do VP_DBG=$d timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_dbg$d.json 2>&1; echo d$d=$?; done

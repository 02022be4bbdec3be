set -x
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 600 python scripts/probe_spread.py c2 > gpurun_out/probe_spread_c2.json 2>&1; echo p2=$?
timeout 900 python scripts/probe_spread.py c5 > gpurun_out/probe_spread_c5.json 2>&1; echo p5=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_spread_strip" -s 1 -c 1 -o gpurun_out/prof_strip_c5g python scripts/one_eval.py c5 0 2 > gpurun_out/ncu_strip_c5.log 2>&1; echo n5=$?

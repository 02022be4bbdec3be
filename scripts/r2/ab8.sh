# own rows default; persistent pair spreader; full GPU suite + bench
set -x
mkdir -p gpurun_out/prof
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_ab8.log 2>&1; echo smoke=$?
VP_PARITY_LOG=gpurun_out/parity_ab8.json timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_ab8.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab8.json 2> gpurun_out/ab8.err; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair" -c 1 -o gpurun_out/prof/full_ab8 python scripts/one_eval.py c5 0 1 > gpurun_out/prof/ncu_full_ab8.log 2>&1; echo ncu=$?

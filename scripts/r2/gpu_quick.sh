# quick check of the current build on a B200: smoke, GPU test suite, default bench line
set -x
D=gpurun_out/${OUT:-q}
mkdir -p $D
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke=$?
VP_PARITY_LOG=$D/parity.json timeout 2400 python -m pytest tests -m gpu -q -s ${PYTEST_K:+-k "$PYTEST_K"} > $D/pytest_gpu.log 2>&1; echo pytest=$?
if [ -z "$SKIP_BENCH" ]; then timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo bench=$?; fi
tail -3 $D/pytest_gpu.log; cat $D/bench_default.json 2>/dev/null | head -c 1500

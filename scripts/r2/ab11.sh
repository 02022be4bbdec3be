# four-step only above n_f = 10000; restriction x with 8 outputs per thread; restriction y with compile-time taps
set -x
mkdir -p gpurun_out/ab11
VP_PARITY_LOG=gpurun_out/ab11/parity.json timeout 2400 python -m pytest tests/test_gpu_parity.py -m gpu -q -s -k "four_step or config3 or config4 or config1 or strip" > gpurun_out/ab11/pytest.log 2>&1; echo pytest=$?
for c in c5 c4 c3; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab11/bench_$c.json 2> gpurun_out/ab11/bench_$c.err; echo bench=$?
done

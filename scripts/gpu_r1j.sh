set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/microbench/fft_prune scripts/microbench/fft_prune.cu -lcufft
./scripts/microbench/fft_prune 23328 5833 > gpurun_out/fft_prune.txt 2>&1; ./scripts/microbench/fft_prune 11340 2836 >> gpurun_out/fft_prune.txt 2>&1; ./scripts/microbench/fft_prune 2744 687 >> gpurun_out/fft_prune.txt 2>&1; echo fftp=$?
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?

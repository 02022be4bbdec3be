# round-2 profiling run: co-bound microbenchmarks, ncu launch list of the default bench (c5), and one
# `ncu --set full` capture per hot kernel of one c5 eval (scripts/one_eval.py)
set -x
mkdir -p gpurun_out/prof
TAG=${TAG:-base}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/microbench/peaks.cu && /tmp/peaks > gpurun_out/prof/microbench_peaks.txt 2>&1; echo peaks=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_peak scripts/microbench/red_peak.cu && /tmp/red_peak >> gpurun_out/prof/microbench_peaks.txt 2>&1
if [ -z "$NO_LAUNCHES" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/prof/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --batch 0 ${BENCH_ARGS} > gpurun_out/prof/ncu_launches_${TAG}.log 2>&1; echo launches=$?
fi
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"${NCU_RE:-k_spread_strip|k_interp_local|k_fft4|k_row4|k_tri_local|k_local_stencil|k_restrict|k_prolong}" \
  -c ${NCU_COUNT:-12} -o gpurun_out/prof/full_${TAG} python scripts/one_eval.py ${CFG:-c5} 0 1 > gpurun_out/prof/ncu_full_${TAG}.log 2>&1; echo ncu=$?

# round-2 evidence run: full GPU test suite, default bench (c5) + reference arm, c2/c3/c4 bench lines,
# co-bound microbenchmarks, ncu launch list (own + cuFFT kernels) and --set full captures of one config-5 eval.
# gpurun returns at most 64 MiB: the full capture is summarised on the box (text / csv) and the report removed.
set -x
D=gpurun_out/${OUT:-ev}
mkdir -p $D
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $D/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke=$?
if [ -z "$SKIP_TESTS" ]; then
VP_PARITY_LOG=$D/parity.json timeout 2700 python -m pytest tests -m gpu -q -s > $D/pytest_gpu.log 2>&1; echo pytest=$?
fi
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo bench=$?
timeout 900 python scripts/bench_layer.py > $D/bench_layer.json 2> $D/bench_layer.err; echo layer=$?
timeout 900 python bench.py --impl reference > $D/bench_ref.json 2> $D/bench_ref.err; echo ref=$?
for c in c2 c3 c4; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > $D/bench_$c.json 2> $D/bench_$c.err; echo bench_$c=$?
done
timeout 900 python bench.py --no-cpu-baseline --batch 0 --opt levels=0 > $D/bench_c5_levels_auto.json 2> $D/bench_c5_levels_auto.err; echo levels=$?
timeout 900 python bench.py --no-cpu-baseline --batch 4 --opt batch_pair=1 > $D/bench_c5_batch_perfield.json 2> $D/bench_c5_batch_perfield.err; echo perfield=$?
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lds_rates scripts/microbench/lds_rates.cu && /tmp/lds_rates > $D/microbench_peaks.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks scripts/microbench/peaks.cu && /tmp/peaks >> $D/microbench_peaks.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/red_peak scripts/microbench/red_peak.cu && /tmp/red_peak >> $D/microbench_peaks.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_|fft|FFT" -c 400 --csv --log-file $D/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --batch 0 > $D/ncu_launches.log 2>&1; echo launches=$?
timeout 1800 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_interp_local|k_fft4|k_row4|k_tri_local|k_local_stencil|k_restrict|k_prolong" \
  -c 20 -o /tmp/prof_c5 python scripts/one_eval.py c5 0 1 > $D/ncu_c5.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_c5.ncu-rep > $D/ncu_c5_summary.txt 2>&1
ncu -i /tmp/prof_c5.ncu-rep --page raw --csv > $D/ncu_c5_raw.csv 2>/dev/null
for k in k_spread_pair k_interp_local k_row4_fwd; do
  ncu -i /tmp/prof_c5.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 --print-source sass > $D/ncu_c5_source_$k.csv 2>/dev/null
done
gzip -f $D/*.csv
du -sh gpurun_out

# round-2 perf iteration: targeted parity tests, c5 bench, optional ncu capture of the spread / interp kernels
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
VP_PARITY_LOG=gpurun_out/parity_perf.json timeout 1500 python -m pytest ${PYTEST_TARGETS} -m gpu -q -s > gpurun_out/pytest_perf.log 2>&1; echo pytest=$?
for c in ${CONFIGS:-c5}; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch ${BATCH:-0} > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo bench_$c=$?
done
if [ -n "$NCU" ]; then
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$NCU" -s ${NCU_SKIP:-6} -c ${NCU_COUNT:-3} \
    -o gpurun_out/prof_${TAG:-x} python bench.py --config ${NCU_CONFIG:-c5} --steps 1 --warmup 3 --no-cpu-baseline --batch 0 \
    > gpurun_out/ncu_${TAG:-x}.log 2>&1; echo ncu=$?
fi

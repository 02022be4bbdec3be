# interpolation tile side A/B at config 5
set -x
mkdir -p gpurun_out/ab13
for t in 64 48 80 96; do
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt interp_tile=$t > gpurun_out/ab13/bench_t$t.json 2> gpurun_out/ab13/bench_t$t.err; echo bench=$?
done

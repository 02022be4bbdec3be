# config 3: level bands with 32-column strips vs row-pair strips
set -x
mkdir -p gpurun_out/ab12
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --batch 0 --opt spread_pack=2 > gpurun_out/ab12/bench_c3_sp2.json 2> gpurun_out/ab12/bench_c3_sp2.err; echo bench=$?
timeout 900 python bench.py --config c3 --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > gpurun_out/ab12/bench_c3.json 2> gpurun_out/ab12/bench_c3.err; echo bench=$?

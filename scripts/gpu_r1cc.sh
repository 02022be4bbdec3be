timeout 600 python bench.py --steps 8 --warmup 3 --config c3 --no-cpu-baseline --batch 0 > gpurun_out/bench_c3_cc.json 2> gpurun_out/bench_c3_cc.err; echo b3=$?

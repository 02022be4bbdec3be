set -x
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --config c5 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench5=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c3 --no-cpu-baseline > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo bench3=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config c4 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench4=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_spread_strip|k_interp_local|k_tri_local12|k_local_stencil" -s 4 -c 4 -o /tmp/prof_c5 python scripts/one_eval.py c5 0 2 > /tmp/ncu_c5.log 2>&1; echo n5=$?
python profiles/ncu_summary.py /tmp/prof_c5.ncu-rep > gpurun_out/ncu_c5_r1final.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_spread_strip|k_interp_local|k_tri_local12|k_local_stencil" -s 4 -c 4 -o /tmp/prof_c4 python scripts/one_eval.py c4 0 2 > /tmp/ncu_c4.log 2>&1; echo n4=$?
python profiles/ncu_summary.py /tmp/prof_c4.ncu-rep > gpurun_out/ncu_c4_r1final.txt 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_spread_strip|k_interp_local|k_band_sum|k_fft" -s 6 -c 8 -o /tmp/prof_c3 python scripts/one_eval.py c3 0 2 > /tmp/ncu_c3.log 2>&1; echo n3=$?
python profiles/ncu_summary.py /tmp/prof_c3.ncu-rep > gpurun_out/ncu_c3_r1final.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file /tmp/launches_c5.csv python scripts/one_eval.py c5 0 2 > /tmp/ncu_launch_c5.log 2>&1; echo l5=$?
gzip -c /tmp/launches_c5.csv > gpurun_out/launches_c5_r1final.csv.gz
du -sh gpurun_out

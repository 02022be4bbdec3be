# two-field pair spreader: ncu capture on config 2 (K = 3: one k_spread_pair2 + one k_spread_pair launch per batch);
# VP_PAIR_WARPS = 8 build against the default on config 5
set -x
D=gpurun_out/ab17
mkdir -p $D
timeout 600 python -m pytest tests/test_gpu_boundary.py -m gpu -q -x > $D/pytest_boundary.log 2>&1; echo pytest=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair" -c 4 -o /tmp/prof_pair2 python scripts/one_eval_batch.py c2 3 > $D/ncu_pair2.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_pair2.ncu-rep > $D/ncu_pair2_summary.txt 2>&1
ncu -i /tmp/prof_pair2.ncu-rep --page source --csv --kernel-name regex:k_spread_pair2 --launch-count 1 --print-source sass > $D/ncu_pair2_source.csv 2>/dev/null
gzip -f $D/ncu_pair2_source.csv
for lib in libvp_w8.so libvp.so; do
VP_LIB=$PWD/paper_2409_11998_b200/$lib timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > $D/bench_$lib.json 2> $D/bench_$lib.err; echo bench=$?
done
tail -3 $D/pytest_boundary.log

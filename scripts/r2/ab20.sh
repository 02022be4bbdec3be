# register budget of the pair spreaders: k_spread_pair2 with 4-warp CTAs x 5 (96 registers) in libvp.so; the
# single-field kernel with the same shape in libvp_s45.so (-DVP_PAIR_WARPS=4 -DVP_PAIR_MINB=5)
set -x
D=gpurun_out/ab20
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch or strip" > $D/pytest.log 2>&1; echo pytest=$?
for lib in libvp.so libvp_s45.so; do
for c in c2 c5; do
VP_LIB=$PWD/paper_2409_11998_b200/$lib timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 4 > $D/bench_${c}_$lib.json 2> $D/bench_${c}_$lib.err; echo bench=$?
done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair" -c 2 -o /tmp/prof_pair2 python scripts/one_eval_batch.py c2 3 > $D/ncu_pair2.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_pair2.ncu-rep > $D/ncu_pair2_summary.txt 2>&1
ncu -i /tmp/prof_pair2.ncu-rep --page source --csv --kernel-name regex:k_spread_pair2 --launch-count 1 --print-source sass > $D/source_pair2.csv 2>/dev/null
python profiles/stall_summary.py $D/source_pair2.csv 30 > $D/stalls_pair2.txt 2>&1
rm -f $D/source_pair2.csv
tail -3 $D/pytest.log
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['phase_ms']['spread'],3), round(d['batch']['ms_per_batch'],3))"; done

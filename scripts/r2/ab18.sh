# two-field pair spreader after removing the 8x unroll: batch bench on c2 and c5, default (two points per
# iteration) against VP_PAIR2_X2=0 (one point per iteration) and the per-field passes (batch_pair=1)
set -x
D=gpurun_out/ab18
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_parity.py -m gpu -q -k "boundary or chunks or polygon or batch or disk or star or lshape" > $D/pytest.log 2>&1; echo pytest=$?
for lib in libvp.so libvp_x1.so; do
for c in c2 c5; do
VP_LIB=$PWD/paper_2409_11998_b200/$lib timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 4 > $D/bench_${c}_$lib.json 2> $D/bench_${c}_$lib.err; echo bench=$?
done
done
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --batch 4 --opt batch_pair=1 > $D/bench_c5_perfield.json 2> $D/bench_c5_perfield.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair" -c 4 -o /tmp/prof_pair2 python scripts/one_eval_batch.py c2 3 > $D/ncu_pair2.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_pair2.ncu-rep > $D/ncu_pair2_summary.txt 2>&1
tail -3 $D/pytest.log
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', d['ms_per_step'], d['batch']['ms_per_batch'])"; done

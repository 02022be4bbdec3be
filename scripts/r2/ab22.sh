# four-field pair spreader (k_spread_pair4): batch tests, K = 4 batch bench on c2 / c5 against pairs only
set -x
D=gpurun_out/ab22
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "batch" > $D/pytest.log 2>&1; echo pytest=$?
for c in c2 c5; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 4 > $D/bench_${c}_quad.json 2> $D/bench_${c}_quad.err; echo bench=$?
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 4 --opt batch_pair=2 > $D/bench_${c}_pairs.json 2> $D/bench_${c}_pairs.err; echo bench=$?
done
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --batch 8 > $D/bench_c5_quad_K8.json 2> $D/bench_c5_quad_K8.err; echo bench=$?
timeout 600 ncu --set full --clock-control none -k regex:"k_spread_pair4" -c 1 -o /tmp/prof_pair4 python scripts/one_eval_batch.py c2 4 > $D/ncu_pair4.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_pair4.ncu-rep > $D/ncu_pair4_summary.txt 2>&1
tail -3 $D/pytest.log
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), d['batch']['K'], round(d['batch']['ms_per_batch'],3))"; done

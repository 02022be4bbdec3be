# interpolation order: targets of a tile dealt to the half-warp groups (default) against rank-major (libvp_deal0.so)
set -x
D=gpurun_out/ab24
mkdir -p $D
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "config1 or config2 or off_node or config3_small or smooth_part" > $D/pytest.log 2>&1; echo pytest=$?
for lib in libvp.so libvp_deal0.so; do
for c in c2 c4 c5; do
VP_LIB=$PWD/paper_2409_11998_b200/$lib timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > $D/bench_${c}_$lib.json 2> $D/bench_${c}_$lib.err; echo bench=$?
done
done
timeout 900 ncu --set full --clock-control none -k regex:"k_interp_local" -c 1 -o /tmp/prof_il python scripts/one_eval.py c5 0 1 > $D/ncu_il.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_il.ncu-rep > $D/ncu_interp_summary.txt 2>&1
tail -3 $D/pytest.log
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); p=d['phase_ms']; print('$f', round(d['ms_per_step'],3), round(p['interp_local'],3))"; done

# pair spreaders with 4-warp CTAs x 4 (128-register cap, libvp_s44.so) against the default 4 x 5 (96 registers)
set -x
D=gpurun_out/ab21
mkdir -p $D
for lib in libvp.so libvp_s44.so; do
for c in c2 c5; do
VP_LIB=$PWD/paper_2409_11998_b200/$lib timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --batch 4 > $D/bench_${c}_$lib.json 2> $D/bench_${c}_$lib.err; echo bench=$?
done
done
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); print('$f', round(d['ms_per_step'],3), round(d['phase_ms']['spread'],3), round(d['batch']['ms_per_batch'],3))"; done

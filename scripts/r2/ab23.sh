# own row FFT passes (k_row4_fwd / k_row4_inv, one CTA per SM): 1024 threads (64-register cap, small spills)
# against 768 (6 warps per sub-partition, 80 registers) and 896 (7, 72 registers) at config 5
set -x
D=gpurun_out/ab23
mkdir -p $D
for t in t768 t896; do
VP_LIB=$PWD/paper_2409_11998_b200/libvp_$t.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "four_step and not fresh" > $D/pytest_$t.log 2>&1; echo pytest_$t=$?
VP_LIB=$PWD/paper_2409_11998_b200/libvp_$t.so timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > $D/bench_$t.json 2> $D/bench_$t.err; echo bench=$?
done
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --batch 0 > $D/bench_t1024.json 2> $D/bench_t1024.err
for t in t768 t896; do tail -1 $D/pytest_$t.log; done
for f in $D/bench_*.json; do python -c "
import json
d=json.load(open('$f')); p=d['phase_ms']; print('$f', round(d['ms_per_step'],3), round(p['fft_fwd'],3), round(p['fft_inv'],3))"; done

# stall reasons of the two north-star kernels at config 5 (one eval under ncu --set full, source page summarised)
set -x
D=gpurun_out/ab19
mkdir -p $D
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair|k_interp_local" -c 2 -o /tmp/prof_ns python scripts/one_eval.py c5 0 1 > $D/ncu.log 2>&1; echo ncu=$?
python profiles/ncu_summary.py /tmp/prof_ns.ncu-rep > $D/ncu_summary.txt 2>&1
for k in k_spread_pair k_interp_local; do
  ncu -i /tmp/prof_ns.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 --print-source sass > $D/source_$k.csv 2>/dev/null
  python profiles/stall_summary.py $D/source_$k.csv 40 > $D/stalls_$k.txt 2>&1
  gzip -f $D/source_$k.csv
done
cat $D/stalls_k_spread_pair.txt | head -20
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_spread_pair2" -c 1 -o /tmp/prof_p2 python scripts/one_eval_batch.py c2 2 > $D/ncu_p2.log 2>&1; echo ncu=$?
ncu -i /tmp/prof_p2.ncu-rep --page source --csv --print-source sass > $D/source_k_spread_pair2.csv 2>/dev/null
python profiles/stall_summary.py $D/source_k_spread_pair2.csv 40 > $D/stalls_k_spread_pair2.txt 2>&1
gzip -f $D/source_k_spread_pair2.csv
timeout 300 python -m pytest tests/test_gpu_boundary.py -m gpu -q > $D/pytest_boundary.log 2>&1; echo pytest=$?
tail -3 $D/pytest_boundary.log

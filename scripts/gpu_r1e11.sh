timeout 1200 ncu --set full --clock-control none -k regex:"k_spread_strip_b" -s 1 -c 1 -o /tmp/prof_b python scripts/one_eval_batch.py c5 4 > /tmp/ncu_b.log 2>&1; echo n=$?
python profiles/ncu_summary.py /tmp/prof_b.ncu-rep > gpurun_out/ncu_c5_batch_r1final.txt 2>&1

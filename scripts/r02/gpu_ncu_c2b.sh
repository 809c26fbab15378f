#!/bin/bash
# c2 evidence: launch list of one training step (libfno kernels) and ncu --set full of every libfno kernel of one
# 1-layer training step, exported on the box to CSV (raw metrics + details page); the report itself stays behind
set -u
O=gpurun_out/r02c2; mkdir -p $O
CMD="python bench.py --config c2 --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
$CMD > $O/plain_c2.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:pass_|b_[xy]|mix_|rowsum|dw_' -s 16 -c 32 --csv --log-file $O/launches_c2.csv $CMD > $O/ncu_launch_c2.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none -k 'regex:pass_|mix_|b_[xy]|rowsum|dw_' -s 16 -c 16 -o /tmp/prof_c2_full $CMD > $O/ncu_full_c2.log 2>&1; echo "ncu full rc=$?"
ncu -i /tmp/prof_c2_full.ncu-rep --page raw --csv > $O/prof_c2_raw.csv 2>&1
ncu -i /tmp/prof_c2_full.ncu-rep --page details --csv > $O/prof_c2_details.csv 2>&1
gzip -f $O/prof_c2_raw.csv $O/prof_c2_details.csv
ls -la $O/

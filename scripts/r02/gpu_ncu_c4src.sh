#!/bin/bash
# ncu --set full with source correlation of the c3 forward pass_c4 launch; the source page (CUDA + SASS, per-line
# stall samples) exported on the box as CSV
set -u
O=gpurun_out/r02src; mkdir -p $O
CMD="python bench.py --config c3 --steps 1 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
$CMD > $O/plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass_c4_kernel" -s 2 -c 1 -o /tmp/prof_c4src $CMD > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_c4src.ncu-rep --page source --csv --print-source cuda,sass > $O/src.csv 2>&1
ncu -i /tmp/prof_c4src.ncu-rep --page raw --csv > $O/raw.csv 2>&1
gzip -f $O/src.csv $O/raw.csv; ls -la $O

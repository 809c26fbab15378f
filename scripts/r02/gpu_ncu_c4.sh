#!/bin/bash
# ncu full capture of the pass_c4 kernels (fwd + bwd) of one layer at a config ($1, default c2)
set -u
CFG=${1:-c2}; TAG=${2:-c4a}
O=gpurun_out/r02; mkdir -p $O
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
$CMD > $O/plain_$TAG.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass_c4" -s 2 -c 2 -o $O/prof_$TAG $CMD > $O/ncu_$TAG.log 2>&1; echo "ncu rc=$?"
tail -3 $O/ncu_$TAG.log

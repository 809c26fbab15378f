#!/bin/bash
# ncu full of the pass C kernels of one layer at a given bench config ($1), tag $2
set -u
CFG=${1:-c3}; TAG=${2:-c3}
mkdir -p gpurun_out
python bench.py --config $CFG --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass_c" -s 2 -c 2 -o gpurun_out/prof_$TAG \
    python bench.py --config $CFG --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"

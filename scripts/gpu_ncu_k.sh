#!/bin/bash
# ncu full (source-level) of the first $3 launches matching kernel regex $1 after skipping $4
set -u
K=${1:-pass_c3}; TAG=${2:-k}; N=${3:-1}; S=${4:-1}
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $S -c $N -o gpurun_out/prof_$TAG \
    python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"

#!/bin/bash
# pass C investigation: ablation table + ncu full (source-level) of one fwd and one bwd pass_c2 launch
set -u
TAG=${1:-pc}
mkdir -p gpurun_out
bash scripts/ablate.sh > gpurun_out/ablate_$TAG.txt 2>&1
cat gpurun_out/ablate_$TAG.txt
python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/plain_$TAG.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"pass_c2" -s 2 -c 2 -o gpurun_out/prof_$TAG \
    python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"

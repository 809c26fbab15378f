#!/bin/bash
# gpu_round.sh, then summarise the ncu capture ON the box and drop the .ncu-rep
# (a full capture of 15 kernels exceeds gpurun's 64 MiB copy-back limit).
set -u
TAG=${1:-r01}
bash scripts/gpu_round.sh "$TAG"
mkdir -p gpurun_out/summary_$TAG && cp profiles/ncu_traffic.json gpurun_out/summary_$TAG/
python scripts/ncu_summary.py --rep gpurun_out/prof_$TAG.ncu-rep --launches gpurun_out/launches_$TAG.csv \
    --out gpurun_out/summary_$TAG --traffic gpurun_out/summary_$TAG/ncu_traffic.json > gpurun_out/summary_$TAG.log 2>&1
echo "summary rc=$?"
rm -f gpurun_out/prof_$TAG.ncu-rep
du -sh gpurun_out

#!/bin/bash
# bench + ncu launch list + ncu full capture of one kernel (regex $1, default pass_c)
set -u
K=${1:-pass_c_kernel}
TAG=${2:-r01}
mkdir -p gpurun_out
python bench.py --steps 20 --warmup 3 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"pass_|b_|mix_|rowsum" -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline \
    > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 2 -c 2 -o gpurun_out/prof_${TAG} \
    python bench.py --steps 2 --warmup 1 --layers 1 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"

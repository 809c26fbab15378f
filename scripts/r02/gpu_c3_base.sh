#!/bin/bash
# round-2 baseline at c3: bench line, ncu launch list, ncu full capture of one training step's kernels
set -u
mkdir -p gpurun_out/r02
O=gpurun_out/r02
python -m paper_2204_01205_b200.build > $O/build.log 2>&1 || { echo build failed; cat $O/build.log; exit 1; }
python bench.py --config c3 --steps 20 --warmup 5 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo "bench c2 rc=$?"
CMD="python bench.py --config c3 --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-graph"
$CMD > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 15 -c 60 --csv --log-file $O/launches_c3.csv $CMD > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -s 15 -c 15 -o $O/prof_c3 $CMD > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"

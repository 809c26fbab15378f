#!/bin/bash
# c3 evidence: launch list of one training step (all libfno kernels), ncu --set full of one launch of each
# libfno kernel of a 1-layer step, then the batched-mixing parity test and B = 1 / 4 / 8 bench lines
set -u
O=gpurun_out/r02; mkdir -p $O
CMD="python bench.py --config c3 --steps 2 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
K='regex:pass_|b_[xy]|mix_|rowsum|dw_'
$CMD > $O/plain_c3.log 2>&1; echo "plain rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -s 15 -c 30 --csv --log-file $O/launches_c3.csv $CMD > $O/ncu_launch_c3.log 2>&1; echo "ncu launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k "$K" -s 15 -c 15 -o $O/prof_c3_full $CMD > $O/ncu_full_c3.log 2>&1; echo "ncu full rc=$?"
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "batched" > $O/pytest_batched.log 2>&1; echo "batched rc=$?"; tail -2 $O/pytest_batched.log
for B in 1 4 8; do
  timeout 600 python bench.py --config c3 --batch $B --layers 1 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c3_B$B.json 2> $O/bench_c3_B$B.err; echo "bench B=$B rc=$?"
done
python scripts/show_bench.py $O/bench_c3_B1.json $O/bench_c3_B4.json $O/bench_c3_B8.json 2>&1 | grep -E "==|mix"

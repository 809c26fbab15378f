#!/bin/bash
# bench lines for the other BASELINE.json configs at N=1 (c3 strong, c4 weak)
mkdir -p gpurun_out
for c in c3 c4; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "bench $c rc=$?"; tail -2 gpurun_out/bench_$c.err
done

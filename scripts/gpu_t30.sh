#!/bin/bash
# T % 4 != 0 tile path: parity (single GPU) + c3 / c2 bench stage times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_network.py -x -q -p no:cacheprovider > gpurun_out/pytest_t30.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_t30.log
for cfg in c3 c2; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_t30_$cfg.json 2>gpurun_out/bench_t30_$cfg.err; echo "bench $cfg rc=$?"
  python scripts/show_bench.py gpurun_out/bench_t30_$cfg.json | grep -E "value|pass_c"
done

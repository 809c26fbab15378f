#!/bin/bash
# first pass_c4 check on the GPU: parity (bounded), group emulation, then c3 / c2 bench lines
set -u
O=gpurun_out/r02; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest_parity.log 2>&1; echo "parity rc=$?"
tail -5 $O/pytest_parity.log
timeout 600 python -m pytest tests/test_gpu_group.py -x -q -m gpu -k "not full_size" > $O/pytest_group.log 2>&1; echo "group rc=$?"
tail -5 $O/pytest_group.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_c4.json 2> $O/bench_c3_c4.err; echo "bench c3 rc=$?"
tail -3 $O/bench_c3_c4.err
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c2_c4.json 2> $O/bench_c2_c4.err; echo "bench c2 rc=$?"

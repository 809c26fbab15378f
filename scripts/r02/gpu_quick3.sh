#!/bin/bash
# quick A/B loop: parity subset (families, split, groups), then the c3 / c2 lines with per-phase times
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-q3}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest_$TAG.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_$TAG.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err; echo "bench c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c2_$TAG.json 2> $O/bench_c2_$TAG.err; echo "bench c2 rc=$?"
python scripts/show_bench.py $O/bench_c3_$TAG.json $O/bench_c2_$TAG.json 2>&1 | grep -E "==|pass_c|bwd.dw "

#!/bin/bash
O=gpurun_out/r02; mkdir -p $O
for ci in 2 3; do FNO_LIB=abl_libs/c4prof.so timeout 300 python scripts/r02/c4_timers.py $ci > $O/c4_timers_c$ci.log 2>&1; echo "c$ci rc=$?"; cat $O/c4_timers_c$ci.log | tail -14; done
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest_t.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_t.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c3_t.json 2> $O/bench_c3_t.err; echo "bench c3 rc=$?"
timeout 300 python bench.py --config c2 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c2_t.json 2> $O/bench_c2_t.err; echo "bench c2 rc=$?"
python scripts/show_bench.py $O/bench_c3_t.json $O/bench_c2_t.json 2>&1 | grep -E "==|pass_c|dominant"

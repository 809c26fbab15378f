#!/bin/bash
O=gpurun_out/r02s; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest.log
for ci in 2 3; do FNO_LIB=abl_libs/c4prof.so timeout 300 python scripts/r02/c4_timers.py $ci fwd > $O/t_c$ci.log 2>&1; echo "timers c$ci rc=$?"; tail -12 $O/t_c$ci.log; done
timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-phases --layers 2 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench c3 rc=$?"
python scripts/show_bench.py $O/bench_c3.json 2>&1 | grep -E "==|pass_c"

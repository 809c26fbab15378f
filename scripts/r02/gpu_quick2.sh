#!/bin/bash
# quick A/B loop: parity subset, then the c3 / c2 lines with per-phase times
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-q2}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_group.py -x -q -m gpu -k "not full_size and not instantiations" > $O/pytest_$TAG.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_$TAG.log
timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err; echo "bench c3 rc=$?"
timeout 300 python bench.py --config c4 --steps 6 --warmup 3 --no-cpu-baseline > $O/bench_c4_$TAG.json 2> $O/bench_c4_$TAG.err; echo "bench c4 rc=$?"
python scripts/show_bench.py $O/bench_c3_$TAG.json $O/bench_c4_$TAG.json 2>&1 | grep -E "==|pass_c|bwd.dw "
python -c "
import json,sys
for f in sys.argv[1:]:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, json.dumps(d['config'].get('pass_c')))
" $O/bench_c3_$TAG.json $O/bench_c4_$TAG.json

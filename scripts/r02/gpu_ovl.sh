#!/bin/bash
# split backward with dw_partial overlapped on a side stream: parity (split + full-size backward), c3 line
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-ovl}
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "split_backward or full_size_backward or families or layer_backward" > $O/pytest_$TAG.log 2>&1; echo "parity rc=$?"; tail -2 $O/pytest_$TAG.log
timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c3_$TAG.json 2> $O/bench_c3_$TAG.err; echo "bench c3 rc=$?"
python scripts/show_bench.py $O/bench_c3_$TAG.json 2>&1 | grep -E "==|pass_c|bwd\.|phases" | head -20
python -c "
import json
d=json.loads(open('$O/bench_c3_$TAG.json').read().strip().splitlines()[-1]); print(json.dumps(d.get('phases')))"

#!/bin/bash
O=gpurun_out/r02; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "batched" > $O/pytest_batched.log 2>&1; echo "batched rc=$?"; tail -2 $O/pytest_batched.log
for B in 1 2 4 8 16; do
  timeout 600 python bench.py --config c3 --batch $B --layers 1 --steps 10 --warmup 3 --no-cpu-baseline --no-phases > $O/bench_c3_B$B.json 2> $O/bench_c3_B$B.err; echo "bench B=$B rc=$?"
  python -c "
import json; d=json.loads(open('$O/bench_c3_B$B.json').read().strip().splitlines()[-1]); s=d['stages']
print('B=$B', 'fwd.mix', s['fwd.mix']['ms_per_step'], 'bwd.mix', s['bwd.mix']['ms_per_step'], 'step', d['ms_per_step'])"
done

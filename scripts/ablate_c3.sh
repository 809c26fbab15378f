#!/bin/bash
# pass_c3 (forward) ablation: stage time with parts skipped (results wrong; timing only)
# bits: 1 phase 2, 2 operand split, 4 epilogue merge/GELU/stores, 16 phase 1
mkdir -p gpurun_out
for a in 0 1 2 4 16 5 3 17 7 23; do
  FNO_ABLATE=$a python bench.py --steps 5 --warmup 3 --layers 1 --no-cpu-baseline > gpurun_out/abl3_$a.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/abl3_$a.json').read().strip().splitlines()[-1]); s=d['stages']
print('ablate=$a', 'fwd.pass_c %.3f' % s['fwd.pass_c']['ms_per_step'])"
done

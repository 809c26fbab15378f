#!/bin/bash
# pass-C ablation: stage times with parts of the kernel skipped (results wrong; timing only)
mkdir -p gpurun_out
for a in 0 1 2 4 8 16 3 7 15 31; do
  FNO_ABLATE=$a python bench.py --steps 5 --warmup 3 --layers 1 --no-cpu-baseline > gpurun_out/abl_$a.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/abl_$a.json').read().strip().splitlines()[-1]); s=d['stages']
print('ablate=$a', 'fwd.pass_c %.3f' % s['fwd.pass_c']['ms_per_step'], 'bwd.pass_c %.3f' % s['bwd.pass_c']['ms_per_step'])"
done

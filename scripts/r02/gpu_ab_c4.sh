#!/bin/bash
# A/B of pass C kernels per config: default library (pass_c4 everywhere) vs FNO_PASS_C4=0 (pass_c2 / pass_c3)
O=gpurun_out/r02; mkdir -p $O
for cfg in c4 c3 c2; do
  timeout 300 python bench.py --config $cfg --steps 6 --warmup 2 --layers 1 --no-cpu-baseline --no-phases > $O/ab_${cfg}_c4.json 2>/dev/null
  FNO_PASS_C4=0 FNO_LIB=abl_libs/knobs.so timeout 300 python bench.py --config $cfg --steps 6 --warmup 2 --layers 1 --no-cpu-baseline --no-phases --allow-dev > $O/ab_${cfg}_old.json 2>&1
  for v in c4 old; do python -c "
import json,sys
try:
  d=json.loads(open('$O/ab_${cfg}_$v.json').read().strip().splitlines()[-1]); s=d['stages']
  print('$cfg $v', 'fwd', s['fwd.pass_c']['ms_per_step'], 'bwd', s['bwd.pass_c']['ms_per_step'], d['config']['pass_c']['fwd']['family'][:8], d['config']['pass_c']['bwd']['family'][:8])
except Exception as e: print('$cfg $v err', e)
"; done
done

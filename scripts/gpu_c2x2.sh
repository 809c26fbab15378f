#!/bin/bash
for i in 1 2; do
  for cfg in ${CFGS:-c2}; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bx.json 2>/dev/null
  echo "== $cfg $i"; python scripts/show_bench.py gpurun_out/bx.json | grep -E "value|pass_c"
  done
done

#!/bin/bash
# A/B of pass C stage times per config: default library vs each abl_libs/*.so
for cfg in ${CFGS:-c2 c3 c4}; do
  for l in default abl_libs/*.so; do
    if [ $l = default ]; then unset FNO_LIB; else export FNO_LIB=$PWD/$l; fi
    timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/abc.json 2>/dev/null
    echo "== $cfg $l $(python scripts/show_bench.py gpurun_out/abc.json | grep -E 'value' | cut -d' ' -f1-2)"
    python scripts/show_bench.py gpurun_out/abc.json | grep -E "pass_c"
  done
done

#!/bin/bash
# A/B: stage times of the default library and each abl_libs/*.so
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab_def.json 2>/dev/null
python scripts/show_bench.py gpurun_out/ab_def.json | grep -E "value|pass_c"
for l in abl_libs/*.so; do
  echo "== $l"
  FNO_LIB=$PWD/$l python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/ab.json 2>/dev/null
  python scripts/show_bench.py gpurun_out/ab.json | grep -E "value|pass_c"
done

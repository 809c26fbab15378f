#!/bin/bash
# A/B of a development library (abl_libs/$1.so) against the default build on the c3 line (same box)
set -u
O=gpurun_out/r02; mkdir -p $O; V=$1
for rep in 1 2; do
  timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline > $O/ab_def_$rep.json 2> /dev/null; echo "def rc=$?"
  FNO_LIB=abl_libs/$V.so timeout 300 python bench.py --config c3 --steps 20 --warmup 5 --no-cpu-baseline --allow-dev > $O/ab_${V}_$rep.json 2> /dev/null; echo "$V rc=$?"
done
python scripts/show_bench.py $O/ab_def_1.json $O/ab_${V}_1.json $O/ab_def_2.json $O/ab_${V}_2.json 2>&1 | grep -E "==|pass_c"

#!/bin/bash
O=gpurun_out/r02t; mkdir -p $O
for ci in 2 3; do for m in fwd bwd; do FNO_LIB=abl_libs/c4prof.so timeout 300 python scripts/r02/c4_timers.py $ci $m > $O/c4_timers_c${ci}_$m.log 2>&1; echo "c$ci $m rc=$?"; tail -13 $O/c4_timers_c${ci}_$m.log; done; done

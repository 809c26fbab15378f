#!/bin/bash
# pass_c4 role timers (development build abl_libs/c4prof.so: scripts/variant_libs.sh c4prof "<c4 TUs> api.cu" -DFNO_C4_PROFILE)
O=gpurun_out/r02t; mkdir -p $O
for ci in ${CONFIGS:-2 3}; do for m in ${MODES:-fwd bwd}; do FNO_LIB=abl_libs/c4prof.so timeout 300 python scripts/r02/c4_timers.py $ci $m > $O/c4_timers_c${ci}_$m.log 2>&1; echo "c$ci $m rc=$?"; tail -13 $O/c4_timers_c${ci}_$m.log; done; done

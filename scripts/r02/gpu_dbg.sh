#!/bin/bash
O=gpurun_out/r02; mkdir -p $O
FNO_LIB=abl_libs/dbg.so timeout 120 python scripts/r02/repro.py > $O/repro_dbg.log 2>&1; echo "dbg rc=$?"; grep -c timeout $O/repro_dbg.log; grep timeout $O/repro_dbg.log | awk '{print $7, $9}' | sort | uniq -c | head -20; tail -3 $O/repro_dbg.log

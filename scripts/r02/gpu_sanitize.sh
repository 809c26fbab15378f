#!/bin/bash
O=gpurun_out/r02; mkdir -p $O
timeout 120 python scripts/r02/repro.py > $O/repro_plain.log 2>&1; echo "plain rc=$?"; tail -3 $O/repro_plain.log
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python scripts/r02/repro.py > $O/sanitize_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "Invalid|ERROR SUMMARY|error|at 0x|ok" $O/sanitize_memcheck.log | head -30

#!/bin/bash
# split backward (pass C family 5): parity, then the per-family A/B at c2 / c3 / c4
set -u
O=gpurun_out/r02; mkdir -p $O; TAG=${1:-split}
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "split_backward or families" > $O/pytest_$TAG.log 2>&1; echo "parity rc=$?"; tail -3 $O/pytest_$TAG.log
for ci in 2 3 4; do timeout 600 python scripts/r02/ab_family.py $ci 2>&1 | grep -E "family|Error"; done | tee $O/ab_$TAG.txt

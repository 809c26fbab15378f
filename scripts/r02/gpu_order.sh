#!/bin/bash
O=gpurun_out/r02o; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "families or forward_matches" > $O/pytest.log 2>&1; echo "parity rc=$?"; tail -1 $O/pytest.log
timeout 600 python scripts/r02/ab_family.py 3 2>&1 | grep "fwd family 4"
CMD="python bench.py --config c3 --steps 1 --warmup 1 --layers 1 --no-cpu-baseline --no-phases --no-graph"
$CMD > $O/plain.log 2>&1 && ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:pass_c4 -c 1 --csv $CMD 2>/dev/null | grep -E "dram__|gpu__time" | cut -d, -f12-

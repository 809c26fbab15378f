#!/bin/bash
O=gpurun_out/r02d; mkdir -p $O
FNO_PEER_EXCHANGE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29611 tests/mp_parity.py --pgrid 4 1 --grid 16 8 16 8 --width 2 --modes 2 2 1 4 --batch 1 --out $O/res.json > $O/dbg4.log 2>&1; echo "rc=$?"
grep -v "^W1019\|elastic" $O/dbg4.log | grep -E "Error|error|Trace|line|assert|FnoError|fno_" | head -30
timeout 1500 python -m pytest tests/test_gpu_multi.py -q -m gpu > $O/pytest_multi4.log 2>&1; echo "multi rc=$?"; tail -2 $O/pytest_multi4.log

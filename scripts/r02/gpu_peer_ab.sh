#!/bin/bash
O=gpurun_out/r02pa; mkdir -p $O
for n in 2 4; do for pe in 1 0; do
  FNO_PEER_EXCHANGE=$pe timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2972$n \
    bench.py --gpus $n --steps 10 --warmup 3 --no-phases --no-cpu-baseline > $O/c3_n${n}_peer$pe.json 2> $O/c3_n${n}_peer$pe.err
  python -c "
import json; d=json.loads(open('$O/c3_n${n}_peer$pe.json').read().strip().splitlines()[-1]); s=d['stages']
print('n=$n peer=$pe', d['ms_per_step'], {k: round(v['ms_per_step'],3) for k,v in s.items() if 'pass_a' in k or 'y_inv' in k or 'exchange' in k})"
done; done

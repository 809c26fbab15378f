#!/bin/bash
# NCCL P2P tuning sweep for the slab exchange at N=2 (exchange stage times)
mkdir -p gpurun_out
run() {
  env "$@" python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 \
    bench.py --gpus 2 --steps 5 --warmup 2 --layers 1 > gpurun_out/nccl_env.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/nccl_env.json').read().strip().splitlines()[-1]); s=d['stages']
print('$*', 'ms/step %.3f' % d['ms_per_step'], ' '.join('%s=%.3f' % (k.split('.')[0][0]+k[-1], v['ms_per_step']) for k, v in s.items() if 'exchange' in k))"
}
run X=1
run NCCL_NCHANNELS_PER_NET_PEER=8
run NCCL_MAX_P2P_NCHANNELS=32 NCCL_NCHANNELS_PER_NET_PEER=16
run NCCL_P2P_NVL_CHUNKSIZE=2097152
run NCCL_MIN_NCHANNELS=32 NCCL_MAX_NCHANNELS=32
run NCCL_PROTO=Simple
run NCCL_P2P_USE_CUDA_MEMCPY=1

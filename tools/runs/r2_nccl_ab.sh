#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
N=${1:-2}
for i in 1 2 3; do
for d in p2p-sm nccl; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --no-cpu --steps 30 --warmup 6 --dense-exchange $d > gpurun_out/r2na.json 2> gpurun_out/r2na.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2na.json').read().strip().splitlines()[-1]); print('N=$N $d', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/r2na.err
done
done

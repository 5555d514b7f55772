#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
for p in "-1,-2,-2" "-2,-1,-2" "-2,0,-2" "-1,-1,-1" "-2,-2,-2"; do
  HP_STREAM_PRIO=$p timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 6 > gpurun_out/r2pr.json 2> gpurun_out/r2pr.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2pr.json').read().strip().splitlines()[-1]); print('prio $p', round(d['ms_per_step']*1e3,1), 'us')" || tail -3 gpurun_out/r2pr.err
done
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --no-cpu --steps 30 --warmup 6 > gpurun_out/r2n4c.json 2> gpurun_out/r2n4c.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2n4c.json').read().strip().splitlines()[-1]); r=d['roofline']; print('N=4 default', round(d['ms_per_step']*1e3,1), 'us K7', round(r['launch_us'],1))" || tail -3 gpurun_out/r2n4c.err
done

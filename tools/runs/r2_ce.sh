#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for d in p2p p2p-sm; do
for w in lm1b lm1b_dense; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 6 --workload $w --dense-exchange $d > gpurun_out/r2ce.json 2> gpurun_out/r2ce.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2ce.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$d $w', round(d['ms_per_step']*1e3,1), 'us K7', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2ce.err
done
done

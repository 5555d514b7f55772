#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/r2d_bench$i.json 2> gpurun_out/r2d_bench$i.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2d_bench$i.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step']*1e3,2), 'us')"
done
timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py lm1b graph 2>&1 | grep spans_us

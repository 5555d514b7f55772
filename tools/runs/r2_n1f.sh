#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
for k in "long_b8=1" "long_b8=2" "long_b8=0"; do
  HP_KNOBS=$k timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/r2i.json 2> gpurun_out/r2i.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2i.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$k', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))"
done
done
HP_KNOBS=long_b8=1 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py lm1b graph 2>&1 | grep spans_us

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for k in "long_b8=1,bcast_tma=1" "long_b8=1,bcast_tma=0" "long_b8=0,bcast_tma=0"; do
echo "== table $k"
HP_KNOBS=$k timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py table graph 2>&1 | grep spans_us
done
for k in "long_b8=1,bcast_tma=0" "long_b8=0,bcast_tma=0" "long_b8=0,bcast_tma=1"; do
  HP_KNOBS=$k timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/r2h.json 2> gpurun_out/r2h.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2h.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$k', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))"
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_multi.py -x -q -k "not lm_consumer" 2>&1 | tail -3
for i in 1 2; do
for s in 1 0; do
for w in lm1b lm1b_sparse; do
  HP_SPLIT_LONG=$s timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 6 --workload $w > gpurun_out/r2sps.json 2> gpurun_out/r2sps.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2sps.json').read().strip().splitlines()[-1]); print('split=$s $w', round(d['ms_per_step']*1e3,1), 'us', d['kernels_us'].get('push:softmax'))" || tail -3 gpurun_out/r2sps.err
done
done
done

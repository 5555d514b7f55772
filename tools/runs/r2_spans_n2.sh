#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for w in lm1b lm1b_sparse; do
  echo "=== $w graph"
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py $w graph 2>&1 | grep -v "^W1019\|OMP_NUM\|\*\*\*\*"
done

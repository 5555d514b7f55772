#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for w in dense table; do
  echo "=== $w graph"
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py $w graph 2>&1 | grep spans_us
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for w in table lm1b; do
  for s in 1 0; do
  echo "=== $w graph split=$s"
  HP_SPLIT_LONG=$s HP_KNOBS=split_long=$s timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py $w graph 2>&1 | grep spans_us
  done
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for w in table table_emb lm1b; do
for b in 1 0; do
echo "== $w b8=$b"
HP_KNOBS=long_b8=$b timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py $w graph 2>&1 | grep spans_us
done
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for kn in "fuse_tree=1" "fuse_tree=0"; do
  echo "== $kn"
  HP_KNOBS=$kn timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29610 tools/span_multi.py lm1b graph 2>&1 | grep spans
  HP_KNOBS=$kn timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 tools/span_multi.py lm1b_sparse graph 2>&1 | grep spans
  HP_KNOBS=$kn timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 tools/span_multi.py table graph 2>&1 | grep spans
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -k "default or p2p-p2p-sm-split or dar_tma" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_emulated.py -q 2>&1 | tail -2
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 > gpurun_out/r2f2b.json 2> gpurun_out/r2f2b.err
tail -1 gpurun_out/r2f2b.json | head -c 300; echo

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
HP_CHECK_OPT=adagrad HP_CHECK_XCHG=p2p HP_CHECK_DENSE=p2p-sm HP_CHECK_DENSE_IN=bf16 HP_CHECK_DENSE_ELEMS=50000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tests/dist_gpu_check.py 2>&1 | grep -v "^W1019" | grep DIST_CHECK
HP_CHECK_OPT=sgd HP_CHECK_XCHG=p2p HP_CHECK_DENSE=nccl HP_CHECK_DENSE_IN=bf16 HP_CHECK_DENSE_ELEMS=50000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 tests/dist_gpu_check.py 2>&1 | grep DIST_CHECK
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "bf16 or dar_buckets or shape" 2>&1 | tail -3

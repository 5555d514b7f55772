#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_parity.py -x -q -k "bf16 or scale_cast or buckets" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "bf16 or dar_buckets or shape" 2>&1 | tail -3

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 600 -p no:cacheprovider \
  > gpurun_out/r2e_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2e_pytest_gpu.txt
tail -n 30 gpurun_out/r2e_pytest_gpu.txt

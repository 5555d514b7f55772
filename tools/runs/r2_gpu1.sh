#!/bin/bash
# round 2, GPU call 1: full -m gpu suite (incl. the emulated multi-rank and
# bench-config parity tests), then a checked N=1 bench line.
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/r2a_gpus.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs --timeout 600 -p no:cacheprovider \
  > gpurun_out/r2a_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2a_pytest_gpu.txt
timeout 600 python bench.py --check --steps 30 --warmup 5 > gpurun_out/r2a_bench_n1.json \
  2> gpurun_out/r2a_bench_n1.err
echo "bench rc=$?" >> gpurun_out/r2a_bench_n1.err
tail -5 gpurun_out/r2a_pytest_gpu.txt
cat gpurun_out/r2a_bench_n1.json | head -c 3000

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for pr in 1 0; do
  echo "== node priority $pr"
  HP_GRAPH_NODE_PRIORITY=$pr timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2961$pr tools/span_multi.py lm1b graph 2>&1 | grep -E "spans|Error|error" | head -5
  HP_GRAPH_NODE_PRIORITY=$pr timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2k_bench_p$pr.json 2>gpurun_out/r2k_bench_p$pr.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2k_bench_p$pr.json').read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step']*1e3, d['kernels_us'])" || tail -5 gpurun_out/r2k_bench_p$pr.err
done

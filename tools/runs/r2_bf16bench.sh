#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for a in "--workload lm1b_dense --dense-in bf16" "--workload lm1b_dense" "--dense-in bf16" ""; do
  n=$(echo "$a" | tr ' -' '__')
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 5 $a > gpurun_out/r2bfb$n.json 2> gpurun_out/r2bfb$n.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2bfb$n.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$a |', round(d['ms_per_step']*1e3,1), 'us', 'K7 graph us', round(r['launch_us'],1), 'bytes', r['algorithmic_bytes'], 'frac', round(r['frac'],3))" || tail -3 gpurun_out/r2bfb$n.err
done

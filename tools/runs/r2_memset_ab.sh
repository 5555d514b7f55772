#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2ms}
for i in 1 2; do
for m in 1 0; do
  HP_KNOBS=plan_memset=$m timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/${T}_m$m.json 2> gpurun_out/${T}_m$m.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_m$m.json').read().strip().splitlines()[-1]); r=d['roofline']
print('memset=$m', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M k4', round(r['launch_us'],1))" || tail -3 gpurun_out/${T}_m$m.err
done
done
for m in 1 0; do
  echo "=== spans memset=$m"
  HP_KNOBS=plan_memset=$m timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py lm1b graph 2>&1 | grep spans_us
done

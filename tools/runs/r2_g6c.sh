#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 300 python bench.py --check > gpurun_out/r2g6c.json 2> gpurun_out/r2g6c.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g6c.json').read().strip().splitlines()[-1]); print('n1 check', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M', d['parity_check']['ok'], d['steps'], d['warmup'])"
for a in "--steps 20 --warmup 5" ""; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu $a > gpurun_out/r2g6n2.json 2> gpurun_out/r2g6n2.err
python -c "
import json; d=json.loads(open('gpurun_out/r2g6n2.json').read().strip().splitlines()[-1]); print('n2 $a', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M', d['config']['steps_per_graph'])" || tail -5 gpurun_out/r2g6n2.err
done

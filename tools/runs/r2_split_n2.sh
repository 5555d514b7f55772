#!/bin/bash
# N=2 full LM1B step vs the dense reduction share of the hot owner (rank 0)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2sp2}
run() {
  name=$1; shift
  timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 5 "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${name}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step']*1e3,1), r['kernel'], 'graph us', round(r['launch_us'],1), 'frac', round(r['frac'],3), flush=True)" || tail -3 gpurun_out/${T}_${name}.err
}
run uni
for s in 0.6,1.4 0.4,1.6 0.2,1.8 0,2 1.4,0.6; do run split_$s --dense-split $s; done

#!/bin/bash
# N=2: K7 (SM stores) scatter / reduce-gather grids, dense-only and full LM1B
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2dg}
run() {
  name=$1; shift; kn=$1; shift
  HP_KNOBS=$kn timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 5 "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${name}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step']*1e3,1), 'graph us', round(r['launch_us'],1), 'frac', round(r['frac'],3), flush=True)" || tail -3 gpurun_out/${T}_${name}.err
}
for g in 0,0 74,0 32,64 64,128 74,148 148,148 148,444; do
  s=${g%,*}; r=${g#*,}
  run dense_${s}_${r} "dar_blocks=$s,dar_rg_blocks=$r" --workload lm1b_dense --dense-exchange p2p-sm
  run full_${s}_${r} "dar_blocks=$s,dar_rg_blocks=$r" --dense-exchange p2p-sm
done

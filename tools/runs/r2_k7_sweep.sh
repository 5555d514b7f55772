#!/bin/bash
# K7 at N=2: raw bidirectional NVLink store/load rate, then the dense-only
# step per transport / scatter grid (graph-timed K7 in the roofline object)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2s}
run() { # name, env knobs, args
  name=$1; shift; kn=$1; shift
  HP_KNOBS=$kn timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 5 "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${name}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step']*1e3,1), r['kernel'], 'graph us', round(r['launch_us'],1), 'eager us', round(r.get('eager_us',0),1), 'frac', round(r['frac'],3), flush=True)" || tail -3 gpurun_out/${T}_${name}.err
}
timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 tools/nvlink_bidir.py 2>&1 | grep rank
for b in 0 148 296 592; do run sm_b$b dar_blocks=$b --workload lm1b_dense --dense-exchange p2p-sm; done
run pipe "" --workload lm1b_dense --dense-exchange p2p-pipe
run pipe_b296 dar_blocks=296 --workload lm1b_dense --dense-exchange p2p-pipe
run nvls "" --workload lm1b_dense --dense-exchange nvls
run pull "" --workload lm1b_dense --dense-exchange p2p-pull

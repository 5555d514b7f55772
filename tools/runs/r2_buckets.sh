#!/bin/bash
# dense buckets: parity (emulated + 2-GPU) then K7 / step timing per bucket count
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2bk}
timeout 900 python -m pytest tests/test_gpu_emulated.py tests/test_gpu_multi.py -x -q -m gpu 2>&1 | tail -5
run() {
  name=$1; shift; kn=$1; shift
  HP_KNOBS=$kn timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 5 "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${name}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step']*1e3,1), r['kernel'][:40], 'graph us', round(r['launch_us'],1), 'eager us', round(r.get('eager_us',0),1), 'frac', round(r['frac'],3), flush=True)" || tail -3 gpurun_out/${T}_${name}.err
}
for b in 1 2 3 4 6; do run dense_b$b dar_buckets=$b --workload lm1b_dense --dense-exchange p2p-sm; done
for b in 1 2 4; do run full_b$b dar_buckets=$b --dense-exchange p2p-sm; done

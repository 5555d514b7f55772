#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 600 python -m pytest tests/test_gpu_emulated.py -x -q -k "tma_scatter" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "dar_rg_tma or dar_tma" 2>&1 | tail -2
for i in 1 2; do
for k in "" "dar_rg_tma=16" "dar_rg_tma=32" "dar_rg_tma=64"; do
for w in lm1b; do
  HP_KNOBS=$k timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu --steps 30 --warmup 6 --workload $w > gpurun_out/r2rg.json 2> gpurun_out/r2rg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2rg.json').read().strip().splitlines()[-1]); r=d['roofline']; print('[$k] $w', round(d['ms_per_step']*1e3,1), 'us K7', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2rg.err
done
done
done

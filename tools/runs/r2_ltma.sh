#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split" 2>&1 | tail -2
for i in 1 2; do
for c in 0 1 2 4 8; do
  HP_KNOBS=long_tma=$c timeout 300 python bench.py --no-cpu --steps 48 --warmup 6 > gpurun_out/r2lt.json 2> gpurun_out/r2lt.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2lt.json').read().strip().splitlines()[-1]); r=d['roofline']; print('long_tma=$c', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2lt.err
done
done
HP_KNOBS=long_tma=2 timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py lm1b graph 2>&1 | grep spans_us

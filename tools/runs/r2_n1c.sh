#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_config.py -x -q 2>&1 | tail -2
for i in 1 2; do
for b in 1 0; do
  HP_KNOBS=long_b8=$b timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/r2f_b$b.json 2> gpurun_out/r2f_b$b.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2f_b$b.json').read().strip().splitlines()[-1]); r=d['roofline']; print('b8=$b', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M k4', round(r['launch_us'],1), round(r['frac'],3))"
done
done
for b in 1 0; do
HP_KNOBS=long_b8=$b timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) tools/span_multi.py lm1b graph 2>&1 | grep spans_us
done

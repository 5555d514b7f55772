#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2 3; do
for c in 0 96 112 128; do
  HP_KNOBS=cbcast=$c timeout 300 python bench.py --no-cpu --steps 48 --warmup 6 > gpurun_out/r2cb.json 2> gpurun_out/r2cb.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2cb.json').read().strip().splitlines()[-1]); r=d['roofline']; print('cbcast=$c', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2cb.err
done
done

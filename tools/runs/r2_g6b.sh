#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for rem in 0 1; do
for a in "--steps 50 --warmup 5" "--steps 60 --warmup 6" "--steps 20 --warmup 5"; do
  HP_BENCH_REMAINDER=$rem timeout 300 python bench.py --no-cpu $a > gpurun_out/r2g6.json 2> gpurun_out/r2g6.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2g6.json').read().strip().splitlines()[-1]); print('rem=$rem $a', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M')" || tail -3 gpurun_out/r2g6.err
done
done

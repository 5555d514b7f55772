#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for a in "--rotations 6 --steps-per-graph 6" "--rotations 12 --steps-per-graph 12" "--rotations 12 --steps-per-graph 6" "--rotations 18 --steps-per-graph 18"; do
for k in "--steps 20 --warmup 5" "--steps 50 --warmup 5"; do
  timeout 300 python bench.py --no-cpu $a $k > gpurun_out/r2g12.json 2> gpurun_out/r2g12.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2g12.json').read().strip().splitlines()[-1]); print('$a $k', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M')" || tail -3 gpurun_out/r2g12.err
done
done

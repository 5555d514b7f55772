#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
for a in "" "" "--no-cpu" ""; do
  timeout 300 python bench.py $a --steps 50 --warmup 5 > gpurun_out/r2v.json 2> gpurun_out/r2v.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2v.json').read().strip().splitlines()[-1]); print('$a', round(d['ms_per_step']*1e3,2), 'us', d['clocks'])"
done

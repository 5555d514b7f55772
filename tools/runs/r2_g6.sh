#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for a in "--steps 20 --warmup 5" "--steps 50 --warmup 5" "--steps 23 --warmup 3" "--check"; do
  timeout 300 python bench.py --no-cpu $a > gpurun_out/r2g6.json 2> gpurun_out/r2g6.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2g6.json').read().strip().splitlines()[-1]); print('$a', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M', d['config']['steps_per_graph'], d.get('parity_check',{}).get('ok'))" || tail -3 gpurun_out/r2g6.err
done

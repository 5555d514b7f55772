#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
for s in 1 2 3; do
  HP_E2E_STREAMS=$s timeout 300 python bench.py --no-cpu --steps 30 --warmup 5 > gpurun_out/r2e2e.json 2> gpurun_out/r2e2e.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2e2e.json').read().strip().splitlines()[-1]); e=d['e2e']; print('streams=$s', '%.4g' % e['value'], 'words/s', 'GB/s %.1f' % (e['h2d_bytes_per_step']*e['value']/2560/1e9))" || tail -3 gpurun_out/r2e2e.err
done
done

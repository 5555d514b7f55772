#!/bin/bash
# N=1 bench lines of the other BASELINE configs with the final defaults
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2cf}
for w in nmt micro_100000 micro_1000000 micro_16000000 dense; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/${T}_$w.json 2> gpurun_out/${T}_$w.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_$w.json').read().strip().splitlines()[-1]); r=d.get('roofline') or {}; c=d.get('cpu_baseline') or {}
print('$w', '%.4g' % d['value'], d['unit'], round(d['ms_per_step']*1e3,1), 'us', 'frac', round(r.get('frac',0),3), 'e2e %.4g' % d['e2e']['value'], 'cpu %.4g' % c.get('value',0))" || tail -3 gpurun_out/${T}_$w.err
done

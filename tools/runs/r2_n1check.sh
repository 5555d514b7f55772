#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2c}
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 300 python bench.py --steps 50 --warmup 5 > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
python -c "
import json; d=json.loads(open('gpurun_out/${T}_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M', 'k4', round(r['launch_us'],1), round(r['frac'],3), 'step frac', round(r['step']['frac'],3), 'e2e', d['e2e']['value'], 'cpu', d['cpu_baseline']['value'], d['clocks'])" || tail -3 gpurun_out/${T}_bench.err

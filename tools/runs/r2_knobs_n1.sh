#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
for k in "" "reduce_bps=4" "reduce_bps=8" "reduce_b=4" "rowstream=1"; do
  HP_KNOBS=$k timeout 300 python bench.py --no-cpu --steps 48 --warmup 6 > gpurun_out/r2kn.json 2> gpurun_out/r2kn.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2kn.json').read().strip().splitlines()[-1]); r=d['roofline']; print('[$k]', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2kn.err
done
done

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
for i in 1 2; do
for g in 1 2 3 6; do
  timeout 300 python bench.py --no-cpu --steps 60 --warmup 6 --steps-per-graph $g > gpurun_out/r2gs.json 2> gpurun_out/r2gs.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2gs.json').read().strip().splitlines()[-1]); print('G=$g', round(d['ms_per_step']*1e3,2), 'us', d['config']['steps_per_graph'], d['config']['rotations'])" || tail -3 gpurun_out/r2gs.err
done
done

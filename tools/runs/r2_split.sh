#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2spl}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_config.py -x -q 2>&1 | tail -3
for i in 1 2; do
for s in 1 0; do
  HP_SPLIT_LONG=$s HP_KNOBS=split_long=$s timeout 300 python bench.py --no-cpu --steps 50 --warmup 5 > gpurun_out/${T}_s$s.json 2> gpurun_out/${T}_s$s.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_s$s.json').read().strip().splitlines()[-1]); r=d['roofline']
print('split=$s', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e6,2), 'M', r['kernel'][:50], 'k4 us', round(r['launch_us'],1), 'frac', round(r['frac'],3), d['kernels_us'])" || tail -3 gpurun_out/${T}_s$s.err
done
done

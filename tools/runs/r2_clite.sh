#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "split or local_apply" 2>&1 | tail -2
for i in 1 2; do
for k in "comb_lite=0" "comb_lite=1" "comb_lite=1,long_tma=2" "comb_lite=1,long_b8=1"; do
  HP_KNOBS=$k timeout 300 python bench.py --no-cpu --steps 48 --warmup 6 > gpurun_out/r2cl.json 2> gpurun_out/r2cl.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2cl.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$k', round(d['ms_per_step']*1e3,2), 'us k4', round(r['launch_us'],1), round(r['frac'],3))" || tail -3 gpurun_out/r2cl.err
done
done

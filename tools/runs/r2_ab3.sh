#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=$1; shift
run() {  # name env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/${T}_$name.json 2>gpurun_out/${T}_$name.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1e3,2), {k:round(v,1) for k,v in d['kernels_us'].items()})" || tail -3 gpurun_out/${T}_$name.err
}
for spec in "$@"; do name=${spec%%:*}; envs=${spec#*:}; run $name ${envs//+/ }; done

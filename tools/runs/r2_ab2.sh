#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
run() {  # name env...
  name=$1; shift
  env "$@" timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu > gpurun_out/r2m_$name.json 2>gpurun_out/r2m_$name.err
  python -c "
import json; d=json.loads(open('gpurun_out/r2m_$name.json').read().strip().splitlines()[-1]); print('$name', round(d['ms_per_step']*1e3,2), {k:round(v,1) for k,v in d['kernels_us'].items()})" || tail -3 gpurun_out/r2m_$name.err
}
run torch HP_STEPGRAPH=0
run torch_inst_lib_launch HP_STEPGRAPH=2
run flags_autofree HP_STEPGRAPH=1 HP_GRAPH_NODE_PRIORITY=0
run flags_autofree_prio HP_STEPGRAPH=9
run flags_upload_prio HP_STEPGRAPH=10
run flags_prio HP_STEPGRAPH=1

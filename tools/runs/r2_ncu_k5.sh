#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-x}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_bcast_rows|k_reduce' -s 40 -c 4 \
    -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu.log 2>&1
echo "rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/${T}_plain.log').read().strip().splitlines()[-1]); print(d['kernels_us'])"

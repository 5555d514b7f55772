#!/bin/bash
# N=1 evidence: launch list of the bench (serialised, cold) + ncu --set full of the
# softmax K4 pair (k_reduce + the long-segment k_bcast_rows) and the dedup cluster kernel
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2}
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_reduce|k_bcast_rows|k_dedup_cluster' -s 60 -c 8 \
    -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu.log 2>&1
echo "full rc=$?"

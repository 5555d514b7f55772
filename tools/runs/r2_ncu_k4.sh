#!/bin/bash
# ncu --set full of the K4 k_reduce launches (softmax + embedding) of a short bench; $1 = tag
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-x}
CMD="python bench.py --steps 2 --warmup 3 --no-cpu"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'k_reduce|k_combine|k_copy_rows' -s 30 -c 6 \
    -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/${T}_ncu.log

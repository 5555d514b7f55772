#!/bin/bash
# final N=1 evidence: GPU suite, checked bench line, ncu launch list, ncu --set full of the K4 pair
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2fin}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rs > gpurun_out/${T}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.txt
tail -3 gpurun_out/${T}_pytest_gpu.txt
timeout 600 python bench.py --check > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
tail -1 gpurun_out/${T}_bench.json | head -c 600; echo
CMD="python bench.py --steps 6 --warmup 3 --no-cpu"
$CMD > gpurun_out/${T}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv \
    --log-file gpurun_out/${T}_launches.csv $CMD > gpurun_out/${T}_launches.log 2>&1
echo "launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:'k_reduce|k_combine|k_bcast_rows|k_dedup_cluster' -s 80 -c 10 \
    -o gpurun_out/${T}_prof $CMD > gpurun_out/${T}_ncu.log 2>&1
echo "full rc=$?"

#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=r2k7
for spec in "default:" "dense_only:--workload lm1b_dense" "nccl_dense:--workload lm1b_dense --dense-exchange nccl"; do
  name=${spec%%:*}; args=${spec#*:}
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus 2 --no-cpu $args > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_${name}.json').read().strip().splitlines()[-1]); r=d['roofline']; print('$name', round(d['ms_per_step']*1e3,1), r['kernel'], 'graph us', round(r['launch_us'],1), 'eager us', round(r.get('eager_us',0),1), 'frac', round(r['frac'],3))" || tail -5 gpurun_out/${T}_${name}.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29655 \
  -m paper_1808_02621_b200.cli tune --graph tools/specs/lm1b_rows.json --cluster tools/specs/box2.json --iterations 20 \
  > gpurun_out/${T}_cli_tune_n2.json 2> gpurun_out/${T}_cli_tune_n2.err
echo "tune rc=$?"; head -c 1200 gpurun_out/${T}_cli_tune_n2.json

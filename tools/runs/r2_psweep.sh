#!/bin/bash
# LM1B step vs partition count P (BASELINE configs[1]: P sweep 8-128), N = $1
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=${1:-2}; T=${2:-r2ps}
for P in 8 16 32 64 128; do
  if [ "$N" = 1 ]; then
    timeout 240 python bench.py --no-cpu --steps 30 --warmup 5 --partitions $P > gpurun_out/${T}_n${N}_p$P.json 2> gpurun_out/${T}_n${N}_p$P.err
  else
    timeout 240 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --no-cpu --steps 30 --warmup 5 --partitions $P > gpurun_out/${T}_n${N}_p$P.json 2> gpurun_out/${T}_n${N}_p$P.err
  fi
  python -c "
import json; d=json.loads(open('gpurun_out/${T}_n${N}_p$P.json').read().strip().splitlines()[-1]); r=d['roofline']; se=d.get('sparse_exchange') or {}
print('N=$N P=$P', round(d['ms_per_step']*1e3,1), 'us', round(d['value']/1e6,2), 'M words/s', r['kernel'][:30], round(r['frac'],3), 'bytes/gpu', se.get('measured_bytes_per_gpu'), flush=True)" || tail -3 gpurun_out/${T}_n${N}_p$P.err
done

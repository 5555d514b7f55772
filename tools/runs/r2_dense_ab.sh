#!/bin/bash
# dense-only K7 A/B on N GPUs: $1 = N, $2 = tag
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=$1; T=$2
run() {
  name=$1; kn=$2; shift 2
  HP_KNOBS=$kn timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N --steps 30 --warmup 5 "$@" \
    > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python - "$T" "$name" <<'PY'
import json,sys
t,n=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/{t}_{n}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(n, "value %.4g" % d["value"], "us %.1f" % (d["ms_per_step"]*1e3), "k7frac", round(r.get("frac",0),3), "k7us", round(r.get("launch_us",0),1), r.get("kernel"))
except Exception as e:
    print(n, "parse failed", e, open(f"gpurun_out/{t}_{n}.err").read()[-800:])
PY
}
run sm_def "" --workload lm1b_dense --dense-exchange p2p-sm
run sm_uni "" --workload lm1b_dense --dense-exchange p2p-sm --dense-split uniform
run sm_296 "dar_blocks=296" --workload lm1b_dense --dense-exchange p2p-sm --dense-split uniform
run sm_592 "dar_blocks=592" --workload lm1b_dense --dense-exchange p2p-sm --dense-split uniform
run nvls "" --workload lm1b_dense --dense-exchange nvls
run full_uni "" --dense-split uniform
run full_nvls "" --dense-exchange nvls

#!/bin/bash
# final multi-GPU evidence on N GPUs: $1 = N, $2 = tag
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
N=$1; T=$2
timeout 1500 python -m pytest tests/test_gpu_multi.py -m gpu -q --timeout 900 -p no:cacheprovider -rs \
  > gpurun_out/${T}_pytest_multi.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_multi.txt
tail -3 gpurun_out/${T}_pytest_multi.txt
run() {
  name=$1; shift
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port $((29700 + RANDOM % 200)) bench.py --gpus $N "$@" \
    > gpurun_out/${T}_bench_${name}.json 2> gpurun_out/${T}_bench_${name}.err
  python - "$T" "$name" <<'PY'
import json,sys
t,n=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/{t}_bench_{n}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    sx=d.get("sparse_exchange") or {}
    print(n, "value %.4g" % d["value"], "us %.1f" % (d["ms_per_step"]*1e3), "k7frac", round(r.get("frac",0),3),
          "e2e %.4g" % d["e2e"]["value"], "clocks", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
except Exception as e:
    print(n, "parse failed", e, open(f"gpurun_out/{t}_bench_{n}.err").read()[-1500:])
PY
}
run default
run nccl --dense-exchange nccl
run sparse_only --workload lm1b_sparse

#!/bin/bash
# tests + bench after a kernel change: $1 = tag
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-x}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider \
  > gpurun_out/${T}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.txt
tail -n 3 gpurun_out/${T}_pytest_gpu.txt
timeout 600 python bench.py --check --steps 30 --warmup 5 > gpurun_out/${T}_bench_n1.json \
  2> gpurun_out/${T}_bench_n1.err
echo "bench rc=$?" >> gpurun_out/${T}_bench_n1.err
python - "$T" <<'PY'
import json,sys
t=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/{t}_bench_n1.json").read().strip().splitlines()[-1])
    r=d["roofline"]
    print("value", d["value"], "ms", d["ms_per_step"], "k4frac", r["frac"], "kern", d["kernels_us"], "step", r["step"], "check", d.get("parity_check"))
except Exception as e:
    print("bench parse failed", e); print(open(f"gpurun_out/{t}_bench_n1.err").read()[-3000:])
PY

#!/bin/bash
# N=1: the GPU suite, then bench lines of every config (default knobs)
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2n1}
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -rs > gpurun_out/${T}_pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.txt
tail -3 gpurun_out/${T}_pytest_gpu.txt
one() {
  name=$1; shift
  timeout 900 python bench.py "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python - "$T" "$name" <<'PY'
import json,sys
t,n=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/{t}_{n}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(n, d["metric"], "%.4g" % d["value"], "us %.1f" % (d["ms_per_step"]*1e3), "k4frac", round(r.get("frac",0),3),
          "k4us", round(r.get("launch_us",0),1), "step frac", round((r.get("step") or {}).get("frac",0),3),
          "e2e %.4g" % d["e2e"]["value"], "cpu", (d.get("cpu_baseline") or {}).get("value"), "check", (d.get("parity_check") or {}).get("ok"))
except Exception as e:
    print(n, "parse failed", e, open(f"gpurun_out/{t}_{n}.err").read()[-1500:])
PY
}
one lm1b --check
one lm1b_b
one nmt --workload nmt
one dense --workload dense
one m100k --workload micro_100000
one m1m --workload micro_1000000 --cpu-steps 1
one m16m --workload micro_16000000 --rotations 2 --cpu-steps 1 --steps 10
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_reference.json 2>&1; tail -1 gpurun_out/${T}_reference.json | head -c 600; echo

#!/bin/bash
# micro config (BASELINE configs[4]: 10M x 128, Zipf 1.1) alpha sweep at N=1, fused vs unfused tree
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=${1:-r2mic}
one() {  # name knobs args...
  name=$1; kn=$2; shift 2
  HP_KNOBS=$kn timeout 900 python bench.py --steps 20 --warmup 3 "$@" > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python - "$T" "$name" <<'PY'
import json,sys
t,n=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/{t}_{n}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(n, d["metric"], "%.4g" % d["value"], "us %.1f" % (d["ms_per_step"]*1e3), "k4frac", round(r.get("frac",0),3),
          "k4us", round(r.get("launch_us",0),1), "U", r.get("unique_rows"), "T", r.get("T"), "cpu", (d.get("cpu_baseline") or {}).get("value"))
except Exception as e:
    print(n, "parse failed", e, open(f"gpurun_out/{t}_{n}.err").read()[-1500:])
PY
}
one m10k_f1 fuse_tree=1 --workload micro_10000
one m100k_f1 fuse_tree=1 --workload micro_100000
one m1m_f1 fuse_tree=1 --workload micro_1000000 --cpu-steps 1
one m1m_f0 fuse_tree=0 --workload micro_1000000 --no-cpu
one m16m_f1 fuse_tree=1 --workload micro_16000000 --rotations 2 --cpu-steps 1
one m16m_f0 fuse_tree=0 --workload micro_16000000 --rotations 2 --no-cpu
one nmt_f1 fuse_tree=1 --workload nmt
one nmt_f0 fuse_tree=0 --workload nmt --no-cpu

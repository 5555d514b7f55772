#!/bin/bash
# A/B of bench lines: $1 = tag, then "name:extra bench args" pairs
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
T=$1; shift
for spec in "$@"; do
  name=${spec%%:*}; extra=${spec#*:}
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu $extra > gpurun_out/${T}_${name}.json 2> gpurun_out/${T}_${name}.err
  python - "$T" "$name" <<'PY'
import json,sys
t,n=sys.argv[1:3]
try:
    d=json.loads(open(f"gpurun_out/{t}_{n}.json").read().strip().splitlines()[-1])
    r=d.get("roofline") or {}
    print(n, "value %.4g" % d["value"], "us %.2f" % (d["ms_per_step"]*1e3), "k4frac", round(r.get("frac",0),3),
          {k: round(v,1) for k,v in d["kernels_us"].items()})
except Exception as e:
    print(n, "parse failed", e, open(f"gpurun_out/{t}_{n}.err").read()[-2000:])
PY
done

line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), (d.get("roofline") or {}).get("frac"), {k: round(v,1) for k,v in (d.get("kernels_us") or {}).items()}) if d else print("FAILED")'; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2 3; do echo "n1: $(timeout 300 python bench.py --no-cpu 2>&1 | line)"; done

line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"], (d.get("roofline") or {}).get("frac"), (d.get("kernels_us") or {})) if d else print("FAILED")'; }
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for i in 1 2; do echo "n1: $(timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu 2>&1 | line)"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_combine -c 20 --csv --log-file gpurun_out/r1d_combine.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1; python tools/launches.py gpurun_out/r1d_combine.csv

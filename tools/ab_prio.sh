run() { HP_STREAM_PRIO=$1 timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu > gpurun_out/prio.log 2>&1; grep '^{' gpurun_out/prio.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1 prio=$1', round(d['ms_per_step']*1e3,2), round(d['value']/1e6,2))"; }
for r in 1 2; do for p in 0,0,0 -1,0,-2 0,0,-2 -2,0,-3 -1,0,-3 -1,-1,-2; do run $p; done; done

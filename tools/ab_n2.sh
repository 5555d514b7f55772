# A/B of instrumentation knobs at N=1 and N=2 (two interleaved repetitions each)
run1() { timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu $1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=1', \"$1\", round(d['ms_per_step']*1e3,2))"; }
run2() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 $1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=2', \"$1\", round(d['ms_per_step']*1e3,2))"; }
for rep in 1 2; do
for k in "--knob rowstream=0 --knob pdl=0" "--knob rowstream=0 --knob pdl=1" "--knob rowstream=1 --knob pdl=1"; do run1 "$k"; done
for k in "--knob rowstream=0 --knob pdl=0 --dense-exchange p2p-sm" "--knob rowstream=0 --knob pdl=1 --dense-exchange p2p-sm" "--knob rowstream=0 --knob pdl=1 --dense-exchange p2p" "--knob rowstream=0 --knob pdl=0 --dense-exchange p2p"; do run2 "$k"; done
done

trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3)) if d else print("FAILED")'; }
b() { local n=$1; local pr=$2; shift 2; local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  echo "n$n prio=$pr $*: $(CUDA_VISIBLE_DEVICES=$dev HP_STREAM_PRIO=$pr timeout 300 bash -c "$(declare -f trun); trun $n $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --no-cpu $*" 2>&1 | line)"; }
for n in 2 4; do
  for pr in "-1,0,-2" "0,-2,-1" "-1,-2,-2" "-2,-1,-2" "0,0,0"; do b $n "$pr"; done
done

trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"]) if d else print("FAILED")'; }
b() { local n=$1; shift; local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  echo "n$n $*: $(CUDA_VISIBLE_DEVICES=$dev timeout 300 bash -c "$(declare -f trun); trun $n $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --no-cpu $*" 2>&1 | line)"; }
echo "== n=1 graph spans lm1b"; CUDA_VISIBLE_DEVICES=0 timeout 200 bash -c "$(declare -f trun); trun 1 29911 tools/span_multi.py lm1b graph" 2>&1 | grep '^{'
b 2 --dense-split 0,1
b 2 --dense-split 1,0
b 2 --dense-split 1,3
b 2 --dense-split 3,1
b 2 --dense-exchange nccl

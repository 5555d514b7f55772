trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,2), d["unit"]) if d else print("FAILED")'; }
b() { local n=$1; shift; local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  echo "n$n $*: $(CUDA_VISIBLE_DEVICES=$dev timeout 300 bash -c "$(declare -f trun); trun $n $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --no-cpu $*" 2>&1 | line)"; }
for n in 2 4; do
  b $n
  b $n --workload lm1b_sparse
  b $n --workload lm1b_sparse --knob owner_stream=0 --knob owner_waves=0
  b $n --knob owner_stream=0 --knob owner_waves=0
  for de in p2p p2p-pipe p2p-sm nccl; do b $n --dense-exchange $de; done
  echo "== n=$n graph spans lm1b"; timeout 200 bash -c "$(declare -f trun); trun $n 2971$n tools/span_multi.py lm1b graph" 2>&1 | grep '^{'
done

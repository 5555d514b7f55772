trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"]) if d else print("FAILED")'; }
b() { local n=$1; shift; local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  echo "n$n $*: $(CUDA_VISIBLE_DEVICES=$dev timeout 300 bash -c "$(declare -f trun); trun $n $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --no-cpu $*" 2>&1 | line)"; }
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "p2p-p2p- or split" 2>&1 | tail -1
echo "single: $(CUDA_VISIBLE_DEVICES=0 timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2 | head -1)"
b 2 --workload lm1b_sparse
b 2
b 4 --workload lm1b_sparse
b 4
echo "== n=2 graph spans table"; CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "$(declare -f trun); trun 2 29904 tools/span_multi.py table graph" 2>&1 | grep '^{'
echo "== n=4 graph spans lm1b"; timeout 200 bash -c "$(declare -f trun); trun 4 29905 tools/span_multi.py lm1b graph" 2>&1 | grep '^{'

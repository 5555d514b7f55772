trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"], d["config"].get("dense_exchange"), d["config"].get("dense_split")) if d else print("FAILED")'; }
b() { local n=$1; shift; local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  CUDA_VISIBLE_DEVICES=$dev timeout 300 bash -c "$(declare -f trun); trun $n $((29500 + RANDOM % 400)) bench.py --gpus $n --steps 30 --warmup 3 --no-cpu $*" > gpurun_out/tmp_b.log 2>&1
  echo "n$n $*: $(cat gpurun_out/tmp_b.log | line)"; grep '^{' gpurun_out/tmp_b.log | tail -1 >> gpurun_out/r1b_multi3.jsonl; }
: > gpurun_out/r1b_multi3.jsonl
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x 2>&1 | tail -2
b 4 --dense-exchange p2p-sm
b 4 --dense-exchange p2p-sm --dense-split uniform
b 4 --dense-exchange p2p --dense-split auto
b 4
b 2
b 2 --workload lm1b_sparse
for w in nmt dense micro_100000; do b 2 --workload $w; b 4 --workload $w; done
echo "== n=4 graph spans lm1b p2p-sm"; timeout 200 bash -c "$(declare -f trun); trun 4 29741 tools/span_multi.py lm1b graph" 2>&1 | grep '^{'

tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
export -f tr
O=gpurun_out/r1b_owner.jsonl; : > $O
run() { local n=$1; shift; local tag=$1; shift
  local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  CUDA_VISIBLE_DEVICES=$dev timeout 240 bash -c "tr $n $((29500 + RANDOM % 400)) $*" > gpurun_out/tmp_${tag}_$n.log 2>&1
  local line=$(grep '^{' gpurun_out/tmp_${tag}_$n.log | tail -1)
  echo "{\"tag\": \"$tag\", \"n\": $n, \"line\": ${line:-null}}" >> $O
}
for k in "owner_stream=2" "owner_stream=1" "owner_stream=0" "owner_stream=2,combine_blocks=32"; do
  echo "single $k: $(CUDA_VISIBLE_DEVICES=0 HP_KNOBS=$k timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2 | tr '\n' ' ')"
done
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_parity.py -q -x > gpurun_out/r1b_owner_tests.log 2>&1; tail -3 gpurun_out/r1b_owner_tests.log
for n in 2 4; do
  run $n full bench.py --gpus $n --steps 30 --warmup 3 --no-cpu
  run $n sparse bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_sparse
  run $n full_pipe bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --dense-exchange p2p-pipe
  run $n full_sm bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --dense-exchange p2p-sm
  run $n full_os1 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --knob owner_stream=1
done
python - <<'PY'
import json
for l in open("gpurun_out/r1b_owner.jsonl"):
    d = json.loads(l); x = d["line"]
    if x: print(d["tag"], d["n"], round(x["ms_per_step"]*1e3, 1), "us", round(x["value"]/1e6, 3), x["unit"])
    else: print(d["tag"], d["n"], "FAILED")
PY

tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
export -f tr
O=gpurun_out/r1b_pipe.jsonl; : > $O
run() { local n=$1; shift; local tag=$1; shift
  local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  CUDA_VISIBLE_DEVICES=$dev timeout 240 bash -c "tr $n $((29500 + RANDOM % 400)) $*" > gpurun_out/tmp_$tag_$n.log 2>&1
  local line=$(grep '^{' gpurun_out/tmp_$tag_$n.log | tail -1)
  echo "{\"tag\": \"$tag\", \"n\": $n, \"line\": ${line:-null}}" >> $O
  [ -z "$line" ] && tail -20 gpurun_out/tmp_$tag_$n.log > gpurun_out/fail_${tag}_$n.log
}
CUDA_VISIBLE_DEVICES=0,1 timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "p2p-pipe" > gpurun_out/r1b_pipe_test.log 2>&1; tail -3 gpurun_out/r1b_pipe_test.log
timeout 600 python -m pytest tests/test_gpu_multi.py -q -x -k "p2p-pipe" > gpurun_out/r1b_pipe_test4.log 2>&1; tail -3 gpurun_out/r1b_pipe_test4.log
if grep -q passed gpurun_out/r1b_pipe_test.log && ! grep -q failed gpurun_out/r1b_pipe_test.log; then
for n in 2 4; do
  run $n dense_pipe bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_dense --dense-exchange p2p-pipe
  run $n dense_pipe_b74 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_dense --dense-exchange p2p-pipe --knob dar_blocks=74
  run $n dense_pipe_b296 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_dense --dense-exchange p2p-pipe --knob dar_blocks=296
  run $n full_pipe bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --dense-exchange p2p-pipe
  run $n full_pipe_b74 bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --dense-exchange p2p-pipe --knob dar_blocks=74
done
fi
python - <<'PY'
import json
for l in open("gpurun_out/r1b_pipe.jsonl"):
    d = json.loads(l); x = d["line"]
    if x: print(d["tag"], d["n"], round(x["ms_per_step"]*1e3, 1), "us", round(x["value"]/1e6, 3), x["unit"])
    else: print(d["tag"], d["n"], "FAILED")
PY

# N=2 / N=4 re-measure on a 4-GPU box: raw NVLink, full step, sparse-only, dense-only per transport, spans
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
export -f tr
O=gpurun_out/r1b_multi.jsonl; : > $O
run() { local n=$1; shift; local tag=$1; shift
  local dev=0,1,2,3; [ $n = 2 ] && dev=0,1
  CUDA_VISIBLE_DEVICES=$dev timeout 240 bash -c "tr $n $((29500 + RANDOM % 400)) $*" > gpurun_out/tmp.log 2>&1
  local line=$(grep '^{' gpurun_out/tmp.log | tail -1)
  echo "{\"tag\": \"$tag\", \"n\": $n, \"line\": ${line:-null}}" >> $O
  [ -z "$line" ] && tail -5 gpurun_out/tmp.log > gpurun_out/fail_$tag_$n.log
}
CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "tr 2 29490 tools/nvlink_bw.py" > gpurun_out/r1b_nvlink_bw.log 2>&1
for n in 2 4; do
  run $n full bench.py --gpus $n --steps 30 --warmup 3 --no-cpu
  run $n sparse bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_sparse
  for de in p2p p2p-sm nccl nvls; do run $n dense_$de bench.py --gpus $n --steps 30 --warmup 3 --no-cpu --workload lm1b_dense --dense-exchange $de; done
  CUDA_VISIBLE_DEVICES=0,1,2,3 timeout 200 bash -c "tr $n 29480 tools/span_multi.py lm1b pipelined" 2>&1 | grep '^{' > gpurun_out/r1b_spans_n$n.jsonl
done
python - <<'PY'
import json
for l in open("gpurun_out/r1b_multi.jsonl"):
    d = json.loads(l); x = d["line"]
    if x: print(d["tag"], d["n"], round(x["ms_per_step"]*1e3, 1), "us", round(x["value"]/1e6, 3), x["unit"])
    else: print(d["tag"], d["n"], "FAILED")
PY
cat gpurun_out/r1b_nvlink_bw.log | grep GB/s

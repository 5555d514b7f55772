# quick iteration loop on a 2-GPU box: parity, single-GPU p2p phase times, N=1 and N=2 bench lines
trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -x 2>&1 | tail -2
for k in "owner_stream=2" "owner_stream=2,owner_waves=0" "owner_stream=0,owner_waves=0"; do
  echo "single $k: $(CUDA_VISIBLE_DEVICES=0 HP_KNOBS=$k timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2 | head -1)"
done
line() { python -c 'import json,sys; d=json.loads([l for l in sys.stdin if l.startswith("{")][-1]); print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,2), d["unit"], "roofline", (d.get("roofline") or {}).get("frac"))'; }
echo "n1 full: $(timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu 2>&1 | line)"
echo "n2 full: $(timeout 300 bash -c "$(declare -f trun); trun 2 29701 bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu" 2>&1 | line)"
echo "n2 sparse: $(timeout 300 bash -c "$(declare -f trun); trun 2 29702 bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu --workload lm1b_sparse" 2>&1 | line)"
echo "== n=2 graph spans table"; timeout 200 bash -c "$(declare -f trun); trun 2 29703 tools/span_multi.py table graph" 2>&1 | grep '^{'

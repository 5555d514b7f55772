trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
for k in "owner_stream=2" "owner_stream=1" "owner_stream=0" "owner_stream=2,combine_blocks=32"; do
  echo "single $k: $(CUDA_VISIBLE_DEVICES=0 HP_KNOBS=$k timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2 | head -1)"
done
for n in 2 4; do
  for wl in table lm1b_sparse lm1b; do
    echo "== n=$n graph spans $wl"
    timeout 200 bash -c "$(declare -f trun); trun $n $((29630+n)) tools/span_multi.py $wl graph" 2>&1 | grep '^{'
  done
done
for b in 444 592; do
  echo "dense pipe n=2 blocks=$b: $(CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "$(declare -f trun); trun 2 2966$((b%10)) bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu --workload lm1b_dense --dense-exchange p2p-pipe --knob dar_blocks=$b" 2>&1 | grep '^{' | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1e3,1))')"
done

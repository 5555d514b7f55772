trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"], d["config"].get("steps_per_graph")) if d else print("FAILED")'; }
for G in 1 2 4; do echo "n1 G=$G: $(CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu --steps-per-graph $G 2>&1 | line)"; done
for G in 1 2 4; do echo "n2 G=$G: $(CUDA_VISIBLE_DEVICES=0,1 timeout 300 bash -c "$(declare -f trun); trun 2 $((29500 + RANDOM % 400)) bench.py --gpus 2 --steps 30 --warmup 3 --no-cpu --steps-per-graph $G" 2>&1 | line)"; done

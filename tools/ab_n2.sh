run2() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 50 --warmup 5 $1 2>&1 | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$NG', \"$1\", round(d['ms_per_step']*1e3,2), round(d['value']/1e6,2))"; }
NG=$(python -c "import torch; print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
for k in "--workload lm1b_dense --dense-exchange nvls" "--workload lm1b_dense --dense-exchange p2p" "--workload lm1b_dense --dense-exchange nccl" "--workload lm1b --dense-exchange nvls" "--workload lm1b --dense-exchange p2p" "--workload lm1b --dense-exchange nccl"; do run2 "$k"; done

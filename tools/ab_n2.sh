run2() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $NG --steps 30 --warmup 3 --no-cpu $1 > gpurun_out/ab_$2.log 2>&1; grep '^{' gpurun_out/ab_$2.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('N=$NG', \"$HP_LIB $1\", round(d['ms_per_step']*1e3,2), round(d['value']/1e6,2), d['e2e']['value']/1e6)"; }
NG=$(python -c "import torch; print(torch.cuda.device_count())")
for i in 1 2 3 4 5; do run2 "" a$i; done
for i in 1 2 3; do run2 "--dense-exchange nvls" n$i; done

# round-1 final measurement set on a 4-GPU box (defaults only)
trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1d_pytest.log 2>&1; tail -2 gpurun_out/r1d_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1d_smoke.log 2>&1; tail -1 gpurun_out/r1d_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/r1d_bench_n1.log 2>&1; tail -1 gpurun_out/r1d_bench_n1.log | cut -c1-300
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --impl reference > gpurun_out/r1d_ref_n1.log 2>&1; tail -1 gpurun_out/r1d_ref_n1.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 timeout 400 bash -c "$(declare -f trun); trun 2 29811 bench.py --gpus 2" > gpurun_out/r1d_bench_n2.log 2>&1; grep '^{' gpurun_out/r1d_bench_n2.log | tail -1 | cut -c1-300
timeout 400 bash -c "$(declare -f trun); trun 4 29812 bench.py --gpus 4" > gpurun_out/r1d_bench_n4.log 2>&1; grep '^{' gpurun_out/r1d_bench_n4.log | tail -1 | cut -c1-300
timeout 400 bash -c "$(declare -f trun); trun 4 29813 bench.py --gpus 4 --impl reference" > gpurun_out/r1d_ref_n4.log 2>&1; grep '^{' gpurun_out/r1d_ref_n4.log | tail -1 | cut -c1-200
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1d_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1d_ncu_launch.log 2>&1; echo "ncu rc=$?"

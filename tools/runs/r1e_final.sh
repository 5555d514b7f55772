trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1e_pytest.log 2>&1; tail -2 gpurun_out/r1e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/r1e_bench_n1.log 2>&1; tail -1 gpurun_out/r1e_bench_n1.log | cut -c1-200
CUDA_VISIBLE_DEVICES=0,1 timeout 400 bash -c "$(declare -f trun); trun 2 29831 bench.py --gpus 2" > gpurun_out/r1e_bench_n2.log 2>&1; grep '^{' gpurun_out/r1e_bench_n2.log | tail -1 | cut -c1-200
timeout 400 bash -c "$(declare -f trun); trun 4 29832 bench.py --gpus 4" > gpurun_out/r1e_bench_n4.log 2>&1; grep '^{' gpurun_out/r1e_bench_n4.log | tail -1 | cut -c1-200

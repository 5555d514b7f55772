# N=2 / N=4 measurement suite (run on a 4-GPU box)
tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
CUDA_VISIBLE_DEVICES=0,1 timeout 300 bash -c "$(declare -f tr); tr 2 29541 bench.py --gpus 2 --steps 30 --warmup 3" 2>&1 | grep '^{' > gpurun_out/r1_bench_n2.json
timeout 300 bash -c "$(declare -f tr); tr 4 29542 bench.py --gpus 4 --steps 30 --warmup 3" 2>&1 | grep '^{' > gpurun_out/r1_bench_n4.json
CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "$(declare -f tr); tr 2 29543 tools/span_multi.py lm1b pipelined" 2>&1 | grep '^{' > gpurun_out/r1_spans_n2.jsonl
timeout 200 bash -c "$(declare -f tr); tr 4 29544 tools/span_multi.py lm1b pipelined" 2>&1 | grep '^{' > gpurun_out/r1_spans_n4.jsonl
timeout 300 bash -c "$(declare -f tr); tr 4 29545 bench.py --gpus 4 --steps 30 --warmup 3 --impl reference" 2>&1 | grep '^{' > gpurun_out/r1_ref_n4.json
for f in gpurun_out/r1_bench_n2.json gpurun_out/r1_bench_n4.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['n_gpus'], round(d['ms_per_step']*1e3,1), round(d['value']/1e6,2), d['config'].get('dense_exchange'), round(d['e2e']['value']/1e6,2))"; done
cat gpurun_out/r1_spans_n2.jsonl gpurun_out/r1_spans_n4.jsonl

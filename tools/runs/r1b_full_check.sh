# full GPU validation on a 4-GPU box + headline lines at N=1/2/4
trun() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
line() { python -c 'import json,sys; L=[l for l in sys.stdin if l.startswith("{")]; d=json.loads(L[-1]) if L else None; print(round(d["ms_per_step"]*1e3,1), "us", round(d["value"]/1e6,3), d["unit"], d["config"].get("dense_exchange"), d["config"].get("dense_split"), (d.get("roofline") or {}).get("frac")) if d else print("FAILED")'; }
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r1c_pytest.log 2>&1; tail -2 gpurun_out/r1c_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "single: $(CUDA_VISIBLE_DEVICES=0 timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2 | head -1)"
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --steps 30 --warmup 3 > gpurun_out/r1c_bench_n1.log 2>&1; echo "n1: $(line < gpurun_out/r1c_bench_n1.log)"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 bash -c "$(declare -f trun); trun 2 29801 bench.py --gpus 2 --steps 30 --warmup 3" > gpurun_out/r1c_bench_n2.log 2>&1; echo "n2: $(line < gpurun_out/r1c_bench_n2.log)"
timeout 300 bash -c "$(declare -f trun); trun 4 29802 bench.py --gpus 4 --steps 30 --warmup 3" > gpurun_out/r1c_bench_n4.log 2>&1; echo "n4: $(line < gpurun_out/r1c_bench_n4.log)"
timeout 300 bash -c "$(declare -f trun); trun 4 29803 bench.py --gpus 4 --steps 5 --warmup 3 --impl reference" > gpurun_out/r1c_ref_n4.log 2>&1; grep '^{' gpurun_out/r1c_ref_n4.log | tail -1 | cut -c1-200
echo "== n=2 graph spans table"; CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "$(declare -f trun); trun 2 29804 tools/span_multi.py table graph" 2>&1 | grep '^{'

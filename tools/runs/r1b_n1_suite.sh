# N=1 re-measure after the k_reduce / stream-priority changes: tests, smoke, bench, ref arm, launches, ncu full
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r1b_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r1b_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1b_smoke.log 2>&1
timeout 300 python bench.py --steps 30 --warmup 3 > gpurun_out/r1b_bench_n1.log 2>&1
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1b_ref_n1.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1b_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1b_ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_reduce --launch-skip 6 -c 2 -o gpurun_out/r1b_k4_full -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1b_ncu_full.log 2>&1
tail -3 gpurun_out/r1b_pytest_gpu.log; tail -1 gpurun_out/r1b_smoke.log; tail -1 gpurun_out/r1b_bench_n1.log; tail -1 gpurun_out/r1b_ref_n1.log

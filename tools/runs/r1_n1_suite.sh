# N=1 measurement suite: bench line, reference arm, launch list, ncu full of K4
set -x
python bench.py --steps 30 --warmup 3 > gpurun_out/r1_bench_n1.log 2>&1
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r1_ref_n1.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reduce --launch-skip 6 -c 2 -o gpurun_out/r1_k4_full -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1_ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:k_copy_rows --launch-skip 6 -c 2 -o gpurun_out/r1_k5_full -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1_ncu_full5.log 2>&1
tail -1 gpurun_out/r1_bench_n1.log; tail -1 gpurun_out/r1_ref_n1.log

# N=1 lines for every BASELINE config (LM1B is the headline; the others are coverage), plus ncu traffic of K4
for w in nmt dense tiny; do timeout 600 python bench.py --workload $w --steps 20 --warmup 3 > gpurun_out/r1b_cfg_${w}_n1.log 2>&1; tail -1 gpurun_out/r1b_cfg_${w}_n1.log | cut -c1-220; done
for w in nmt dense; do timeout 600 python bench.py --impl reference --workload $w --steps 2 --warmup 3 > gpurun_out/r1b_ref_${w}_n1.log 2>&1; tail -1 gpurun_out/r1b_ref_${w}_n1.log | cut -c1-200; done
for d in 1000 10000 100000 1000000; do timeout 600 python bench.py --workload micro_$d --steps 20 --warmup 3 --no-cpu > gpurun_out/r1b_cfg_micro_${d}_n1.log 2>&1; tail -1 gpurun_out/r1b_cfg_micro_${d}_n1.log | cut -c1-200; done
timeout 600 ncu --set full --clock-control none -k regex:"k_reduce|k_combine" --launch-skip 8 -c 4 -o gpurun_out/r1b_k4_traffic -f python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r1b_k4_traffic.log 2>&1; tail -1 gpurun_out/r1b_k4_traffic.log

tr() { python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port $2 "${@:3}"; }
CUDA_VISIBLE_DEVICES=0,1 timeout 200 bash -c "$(declare -f tr); tr 2 29471 tools/nvlink_bidir.py" 2>&1 | grep rank
timeout 200 bash -c "$(declare -f tr); tr 4 29472 tools/nvlink_bidir.py" 2>&1 | grep rank
CUDA_VISIBLE_DEVICES=0 timeout 200 python tools/p2p_single.py 5 time 2>&1 | tail -2
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_owner|k_reduce|k_combine|k_copy" --launch-skip 8 -c 4 -o gpurun_out/r1b_p2p_single -f python tools/p2p_single.py 5 > gpurun_out/r1b_p2p_single_ncu.log 2>&1; tail -2 gpurun_out/r1b_p2p_single_ncu.log

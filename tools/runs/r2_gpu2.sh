#!/bin/bash
cd "$GRAFT_REPO_ROOT" || exit 1
mkdir -p gpurun_out
export HP_WAIT_TIMEOUT_CYCLES=400000000
(timeout 120 python tools/emu_diag.py basic) > gpurun_out/r2b_diag_lazy.txt 2>&1
(CUDA_MODULE_LOADING=EAGER timeout 180 python tools/emu_diag.py basic) > gpurun_out/r2b_diag_eager.txt 2>&1
(timeout 120 python tools/emu_diag.py pipe) > gpurun_out/r2b_diag_pipe.txt 2>&1
(timeout 300 compute-sanitizer --tool memcheck python tools/emu_diag.py ce) > gpurun_out/r2b_diag_ce_memcheck.txt 2>&1
tail -n 12 gpurun_out/r2b_diag_*.txt

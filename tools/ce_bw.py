"""Copy-engine (cudaMemcpyPeerAsync) NVLink bandwidth between GPU 0 and 1.

python tools/ce_bw.py  -> one line per size: uni- and bidirectional GB/s.
"""
import torch

assert torch.cuda.device_count() >= 2
d0, d1 = torch.device("cuda:0"), torch.device("cuda:1")
for mb in (4, 19, 38, 76):
    n = mb * (1 << 20) // 4
    a0, b0 = torch.randn(n, device=d0), torch.empty(n, device=d0)
    a1, b1 = torch.randn(n, device=d1), torch.empty(n, device=d1)
    s0, s1 = torch.cuda.Stream(d0), torch.cuda.Stream(d1)
    res = {}
    for mode in ("uni", "bi"):
        for _ in range(3):
            with torch.cuda.stream(s0):
                b1.copy_(a0, non_blocking=True)
            if mode == "bi":
                with torch.cuda.stream(s1):
                    b0.copy_(a1, non_blocking=True)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        reps = 10
        with torch.cuda.device(d0):
            e[0].record(s0)
        with torch.cuda.device(d1):
            e[2].record(s1)
        for _ in range(reps):
            with torch.cuda.stream(s0):
                b1.copy_(a0, non_blocking=True)
            if mode == "bi":
                with torch.cuda.stream(s1):
                    b0.copy_(a1, non_blocking=True)
        with torch.cuda.device(d0):
            e[1].record(s0)
        with torch.cuda.device(d1):
            e[3].record(s1)
        torch.cuda.synchronize(d0); torch.cuda.synchronize(d1)
        t = e[0].elapsed_time(e[1]) / reps * 1e-3
        res[mode] = round(n * 4 / t / 1e9, 1)
        if mode == "bi":
            t1 = e[2].elapsed_time(e[3]) / reps * 1e-3
            res["bi_other"] = round(n * 4 / t1 / 1e9, 1)
    print({"MB": mb, "GBps_per_direction": res}, flush=True)

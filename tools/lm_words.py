"""Training words/s of the LM consumer (paper_1808_02621_b200.lm.HybridLM) at
LM1B shapes on one GPU: pull -> LSTM + sampled softmax fwd/bwd -> hybrid step."""
import json, sys
import torch
sys.path.insert(0, '.')
from paper_1808_02621_b200.lm import HybridLM

lm = HybridLM(device="cuda:0")
batches = [lm.batch_ids() for _ in range(4)]
for i in range(5):
    lm.step(*batches[i % 4])
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
K = 30
a.record()
losses = [lm.step(*batches[i % 4]) for i in range(K)]
b.record()
torch.cuda.synchronize()
us = a.elapsed_time(b) * 1e3 / K
print(json.dumps({"what": "LM1B-shaped training step with a real consumer (N=1)",
                  "us_per_step": us, "words_per_s": lm.batch * lm.seq / (us * 1e-6),
                  "dense_params": lm.n_dense, "loss_first": losses[0], "loss_last": losses[-1]}))

"""A real consumer of the hybrid step: an LM1B-style
language model whose embedding and sampled-softmax tables are the sharded
sparse Weights and whose LSTM is the dense Weight.

One training step of one worker (one process per GPU; N=1 keeps every
partition local — the reference marks all Weights AR at one machine,
`placement.py:111` — N>1 shards the tables across the box):

1. pull: the token rows and the softmax rows (targets + shared log-uniform
   samples) are looked up with :meth:`HybridRunner.pull` — a local gather at
   N=1, NVLink reads from each row's owner slab at N>1 (`hp_xchg_pull`);
2. compute: embedding rows → LSTM (cuDNN, PyTorch plumbing) → sampled softmax
   cross entropy; backward gives IndexedSlices for both tables (one gradient
   row per looked-up position) and dense LSTM gradients;
3. :meth:`HybridRunner.step` dedups, reduces and applies the sparse gradients
   with the sparse optimizer (Adagrad) and averages the dense gradient (K7);
   the averaged dense gradient updates the LSTM with plain SGD.

``words/s`` here includes the model's own compute — the synthetic-gradient
bench (`bench.py`) measures the communication/update path alone.
"""

from __future__ import annotations

import json

import numpy as np
import torch

from . import ops
from .model import ClusterSpec, load_graph_spec
from .placement import transform_hybrid
from .synth import log_uniform_ids, zipf_ids


class HybridLM:
    def __init__(self, V: int = 800_000, D: int = 512, hidden: int = 1024, batch: int = 128,
                 seq: int = 20, samples: int = 8192, partitions: int = 8, lr: float = 0.2,
                 dense_lr: float = 0.05, device="cuda", seed: int = 0, rank: int = 0,
                 world_size: int = 1, comm=None):
        from .runner import HybridRunner

        self.V, self.D, self.batch, self.seq, self.samples = V, D, batch, seq, samples
        self.device = torch.device(device)
        torch.manual_seed(seed)
        self.lstm = torch.nn.LSTM(D, hidden, batch_first=True).to(self.device)
        self.proj = torch.nn.Linear(hidden, D, bias=False).to(self.device)
        self.dense_params = list(self.lstm.parameters()) + list(self.proj.parameters())
        n_dense = sum(p.numel() for p in self.dense_params)
        self.n_dense = n_dense + (-n_dense) % 4
        T = batch * seq
        graph = load_graph_spec(json.dumps({
            "name": "lm", "batch_per_gpu": batch, "compute_us_per_gpu": 0.0,
            "variables": [
                {"name": "lstm", "elements": self.n_dense, "elem_bytes": 4, "alpha": 1,
                 "kind": "dense"},
                {"name": "embedding", "elements": V, "elem_bytes": 4 * D,
                 "alpha": min(1.0, T / V), "kind": "sparse", "partitionable": True},
                {"name": "softmax", "elements": V, "elem_bytes": 4 * D,
                 "alpha": min(1.0, (T + samples) / V), "kind": "sparse", "partitionable": True}]}))
        cluster = ClusterSpec.b200_box(world_size)
        plan = transform_hybrid(graph, cluster,
                                partitions={"embedding": partitions, "softmax": partitions})
        self.runner = HybridRunner(plan, graph, cluster, device=self.device, seed=seed,
                                   rank=rank, world_size=world_size, comm=comm,
                                   optimizer=ops.OptimizerConfig("adagrad", lr=lr))
        self.dense_lr = dense_lr
        self.rng = np.random.default_rng(seed * 1000 + rank)  # each worker its own data
        self._flat = torch.zeros(self.n_dense, device=self.device)

    def batch_ids(self):
        """Zipf(1.1) token ids [batch, seq+1] (inputs and next-token targets) and
        the step's shared log-uniform softmax samples."""
        toks = zipf_ids(self.rng, self.V, self.batch * (self.seq + 1)).reshape(self.batch, -1)
        samp = log_uniform_ids(self.rng, self.V, self.samples)
        return (torch.from_numpy(toks).to(self.device), torch.from_numpy(samp).to(self.device))

    def _pull(self, name: str, ids: torch.Tensor) -> torch.Tensor:
        return self.runner.pull(name, ids.contiguous())

    def step(self, toks: torch.Tensor, samp: torch.Tensor) -> float:
        inp, tgt = toks[:, :-1].reshape(-1), toks[:, 1:].reshape(-1)
        sm_ids = torch.cat([tgt, samp])
        emb = self._pull("embedding", inp).requires_grad_(True)            # [T, D]
        w_sm = self._pull("softmax", sm_ids).requires_grad_(True)          # [T + S, D]
        h, _ = self.lstm(emb.view(self.batch, self.seq, self.D))
        h = self.proj(h.reshape(-1, h.shape[-1]))                           # [T, D]
        T = h.shape[0]
        true_logit = (h * w_sm[:T]).sum(-1, keepdim=True)                   # [T, 1]
        samp_logit = h @ w_sm[T:].t()                                       # [T, S]
        logits = torch.cat([true_logit, samp_logit], dim=1)
        loss = torch.nn.functional.cross_entropy(logits, torch.zeros(T, dtype=torch.long,
                                                                     device=self.device))
        for p in self.dense_params:
            p.grad = None
        loss.backward()
        off = 0
        for p in self.dense_params:  # the dense Weight's gradient, flat
            n = p.numel()
            self._flat[off:off + n].copy_(p.grad.reshape(-1))
            off += n
        self.runner.step({"embedding": (inp.contiguous(), emb.grad.contiguous()),
                          "softmax": (sm_ids.contiguous(), w_sm.grad.contiguous()),
                          "lstm": self._flat}, timed=False)
        g = self.runner.dense_out["lstm"]
        off = 0
        with torch.no_grad():
            for p in self.dense_params:
                n = p.numel()
                p.add_(g[off:off + n].view_as(p), alpha=-self.dense_lr)
                off += n
        return float(loss.detach())

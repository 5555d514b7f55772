"""a real model consumes the hybrid step (HybridLM, N=1):
pulled rows feed an LSTM + sampled softmax, its IndexedSlices and dense LSTM
gradients go back through HybridRunner.step."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def test_lm_trains_through_the_hybrid_step():
    from paper_1808_02621_b200.lm import HybridLM

    lm = HybridLM(V=50_000, D=128, hidden=256, batch=16, seq=10, samples=512, partitions=4,
                  device="cuda:0", seed=3)
    emb0 = lm.runner.tables["embedding"].w.clone()
    toks, samp = lm.batch_ids()
    losses = [lm.step(toks, samp) for _ in range(8)]  # the same batch: the loss must fall
    torch.cuda.synchronize()
    assert all(np.isfinite(losses)), losses
    assert losses[-1] < losses[0], losses
    touched = torch.unique(toks[:, :-1].reshape(-1))
    w = lm.runner.tables["embedding"].w
    assert not torch.equal(w[touched], emb0[touched])          # touched rows updated
    untouched = torch.ones(w.shape[0], dtype=torch.bool, device=w.device)
    untouched[touched] = False
    assert torch.equal(w[untouched], emb0[untouched])          # only touched rows

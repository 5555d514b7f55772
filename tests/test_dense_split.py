"""Host logic of the dense reduction split (HybridRunner._dense_split_weights):
which ranks get no dense reduction chunk. Runs on CPU (no device objects)."""

import json
from types import SimpleNamespace

import pytest

import paper_1808_02621_b200 as hp
from paper_1808_02621_b200.runner import HybridRunner
from paper_1808_02621_b200.synth import WORKLOADS


def _fake(n, dense_exchange="p2p-sm"):
    graph = hp.load_graph_spec(json.dumps(WORKLOADS["lm1b"].graph_json()))
    cluster = hp.ClusterSpec.b200_box(n)
    plan = hp.transform_hybrid(graph, cluster, partitions={"embedding": 8, "softmax": 8})
    return SimpleNamespace(world_size=n, plan=plan, graph=graph, dense_exchange=dense_exchange)


@pytest.mark.parametrize("n", [4, 8])
def test_auto_zeroes_partition0_owners(n):
    f = _fake(n)
    w = HybridRunner._dense_split_weights(f, "auto")
    hot = {f.plan.owner_of("embedding", 0), f.plan.owner_of("softmax", 0)}
    assert w == [0.0 if r in hot else 1.0 for r in range(n)]
    assert sum(w) > 0


def test_auto_uniform_below_four_ranks_and_for_pipe():
    assert HybridRunner._dense_split_weights(_fake(2), "auto") is None
    assert HybridRunner._dense_split_weights(_fake(4, "p2p-pipe"), "auto") is None
    assert HybridRunner._dense_split_weights(_fake(4), "uniform") is None


def test_explicit_weights_checked():
    assert HybridRunner._dense_split_weights(_fake(4), [1, 2, 3, 4]) == [1, 2, 3, 4]
    with pytest.raises(ValueError):
        HybridRunner._dense_split_weights(_fake(4), [1, 2])
    with pytest.raises(ValueError):
        HybridRunner._dense_split_weights(_fake(4), "bogus")

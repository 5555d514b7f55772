"""B200-native hybrid communication (Parallax, arXiv 1808.02621).

Drop-in for the reference package ``sparseplan`` on the hybrid-communication
path: the planner names (Weight classification, partitioning, placement, the
P search) keep the reference's signatures and semantics, and
:class:`HybridRunner` replaces the simulated iteration with real sm_100a
kernels + NCCL over NVLink. Device modules (``runner``, ``ops``, ``comm``)
import torch and the CUDA library lazily so the planner works without a GPU.
"""

from .model import (
    ClusterSpec,
    GraphSpec,
    PartitionSet,
    SpecError,
    SpecParseError,
    VariableSpec,
    even_split,
    load_cluster_spec,
    load_graph_spec,
    model_alpha,
    partition_bounds,
    partition_of_row,
    partition_variable,
    shard_count,
)
from .placement import (
    DistributedPlan,
    Mechanism,
    MechanismPolicy,
    PlacedNode,
    assign_mechanism,
    plan_from_dict,
    plan_to_dict,
    transform_ar,
    transform_hybrid,
    transform_ps,
    validate_plan,
)
from .stats import ComputeProfile, IterationStats, Message, TransferReport
from .transfer import payload_transfer, transfer_model
from .tuning import (
    CostModelParams,
    TuneResult,
    TuningError,
    fit_theta,
    optimal_p,
    predict_time,
    sample_search,
    tune,
    tune_evaluator,
)

__version__ = "0.1.0"

_LAZY = {
    "HybridRunner": ("runner", "HybridRunner"),
    "ShardedTable": ("runner", "ShardedTable"),
    "device_evaluator": ("runner", "device_evaluator"),
    "simulate_training": ("runner", "simulate_training"),
    "OptimizerConfig": ("ops", "OptimizerConfig"),
    "Comm": ("comm", "Comm"),
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod, attr = _LAZY[name]
        return getattr(importlib.import_module(f".{mod}", __name__), attr)
    raise AttributeError(name)

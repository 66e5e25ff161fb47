"""B200-native spatiotemporal Hawkes log-likelihood + gradient engine.

The hot path of arxiv 2407.11349 (the O(N^2) StHP likelihood that drives
every MCMC step of the cut-posterior sampler) as hand-written sm_100a CUDA
behind a C ABI (include/hawkes_b200.h).  This package is the thin Python
mirror of the reference's interface; see DESIGN.md.
"""
from .engine import (Catalog, Evaluator, HawkesParams, LikelihoodWorkspace, Partition, Precision, Region, Regions,
                     Variant, benchmark_catalog, event_contribution, log_likelihood,
                     log_likelihood_and_gradient, make_partition, plan_shards)

__all__ = [
    "Region", "Regions",
    "Catalog", "Evaluator", "HawkesParams", "LikelihoodWorkspace", "Partition", "Precision",
    "Variant", "benchmark_catalog", "event_contribution", "log_likelihood",
    "log_likelihood_and_gradient", "make_partition", "plan_shards",
]

"""Garfield (arXiv 2010.05888) GAR hot path, B200-native.

The paper's aggregation interface (§4.1): ``init(name, n,
f)`` then ``aggregate(tensors)``; the device follows the inputs.  Here every
step runs in the sm_100a kernels of ``libgar.so`` (C ABI: include/gar.h);
this package only marshals arguments.

    g = paper_2010_05888_b200.init("bulyan", n=31, f=7)
    out = g.aggregate(list_of_cuda_fp32_tensors)      # fp32[d] (bf16 inputs too: widened exactly)
    idx = g.select(list_of_cuda_fp32_tensors)         # int32 indices (Krum family)
"""
from ._lib import (GarError, RULES, gar_aggregate, gar_aggregate_ex, gar_combine, gar_distances,  # noqa: F401
                   gar_gram_partial, gar_num_selected, gar_check_args, gar_select, gar_select_from_gram, gar_status_string,
                   gar_last_error, gar_gram_exchange,
                   gar_aggregate_bcast, gar_combine_bcast, gar_aggregate_mcast, gar_combine_mcast,
                   gar_trimmed_membership, gar_aggregate_sgd, gar_combine_sgd, gar_nonfinite_rows,
                   gar_workspace_bytes, gar_aggregate_dt, gar_select_dt, gar_distances_dt,
                   gar_gram_partial_dt, gar_combine_dt)
from .gar import Aggregator, TooManyNonFinite, aggregate_sanitized, init, sanitize  # noqa: F401

__all__ = ["init", "Aggregator", "GarError", "RULES", "gar_aggregate", "gar_aggregate_ex", "gar_select",
           "gar_distances", "gar_gram_partial", "gar_select_from_gram", "gar_combine", "gar_workspace_bytes",
           "gar_num_selected", "gar_check_args", "gar_status_string", "gar_last_error", "gar_aggregate_bcast", "gar_combine_bcast",
           "gar_aggregate_mcast", "gar_combine_mcast", "gar_trimmed_membership", "gar_aggregate_sgd",
           "gar_combine_sgd", "gar_nonfinite_rows", "sanitize", "aggregate_sanitized", "TooManyNonFinite",
           "gar_aggregate_dt", "gar_select_dt", "gar_distances_dt", "gar_gram_partial_dt", "gar_combine_dt"]

"""B200-native FiGaRo hot path (arXiv 2204.00525): the QR factor R of a
natural join, computed on the GPU without materialising the join.

The compute path is libfigaro_cuda.so (C ABI in include/figaro_cuda.h,
sources in csrc/).  This package is its Python host mirror of the reference
API (see figaro.py) plus the synthetic workloads used by bench.py.
"""
from .figaro import (  # noqa: F401
    Context, JoinTree, Layout, NodeCounts, OutSpan, PipelineOptions,
    PipelineResult, Relation, TriangularFactor, build_join_tree, empty_join_error,
    error, get_context, group_keys, heads_tails, integrity_error, make_layout,
    parse_error, rank_error, run_pipeline, schema_error, size_error, tree_error,
    tsqr, unsupported_error,
)

__all__ = [
    "Context", "JoinTree", "Layout", "NodeCounts", "OutSpan", "PipelineOptions",
    "PipelineResult", "Relation", "TriangularFactor", "build_join_tree",
    "empty_join_error", "error", "get_context", "group_keys", "heads_tails",
    "integrity_error", "make_layout", "parse_error", "rank_error", "run_pipeline",
    "schema_error", "size_error", "tree_error", "tsqr", "unsupported_error",
]

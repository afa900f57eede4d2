"""sparselex-b200: B200-native eager sparse BM25 scoring (BM25S hot path, arXiv 2407.03618).

Public API mirrors the reference SPEC (build_index / score_query / top_k / retrieve /
retrieve_batch); everything computes through libsparselex_b200.so (CUDA sm_100a).
"""
from .api import (BM25Params, Comm, QueryResult, SearchIndex, Variant, build_index, is_sparse_variant, load_index, merge_candidates, retrieve,
                  retrieve_batch, retrieve_local, score_query, shard_ranges, top_k)

__all__ = ["BM25Params", "Comm", "QueryResult", "SearchIndex", "Variant", "build_index", "is_sparse_variant", "load_index",
           "merge_candidates", "retrieve", "retrieve_batch", "retrieve_local", "score_query", "shard_ranges", "top_k"]

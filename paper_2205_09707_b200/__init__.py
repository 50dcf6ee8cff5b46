"""B200-native PLAID four-stage search (drop-in for the reference `lir` searcher).

The engine is libplaid.so (CUDA sm_100a kernels + C++ host + C ABI,
include/plaid.h); this package is the Python mirror of the reference's
interface over that ABI, plus the host-side index container and the
deterministic synthetic index generator used by tests and the bench.
"""
from .api import (BatchSearcher, MultiGpuSearcher, build_index, CandidateSet, DeviceIndex, ErrorCode, PlaidError, ScoreMode, SearchOptions,
                  SearchParams, SearchResult, Searcher, StageTrace, default_params_for_k,
                  checksum, encode_corpus, lut_build, pack_residual, save_index, search, stage3_width, validate_params,
                  validate_query)
from .hostindex import (HostIndex, build_inverted_list, fnv_digest, generate_index, generate_queries,
                        load_index_host, quantizer)

__all__ = [
    "CandidateSet", "DeviceIndex", "ErrorCode", "PlaidError", "ScoreMode", "SearchOptions",
    "BatchSearcher", "MultiGpuSearcher", "build_index", "SearchParams", "SearchResult", "Searcher", "StageTrace", "default_params_for_k", "lut_build",
    "pack_residual", "search", "stage3_width", "validate_params", "validate_query", "HostIndex",
    "build_inverted_list", "generate_index", "generate_queries", "quantizer", "save_index", "checksum", "encode_corpus",
    "fnv_digest", "load_index_host",
]

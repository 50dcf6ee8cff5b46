"""ctypes binding of libplaid.so (include/plaid.h).

The product path is the CUDA library; there is no CPU fallback.  Loading fails
loudly when the in-tree build is missing.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_LIB_DIR = Path(__file__).resolve().parent / "_lib"

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
f32p = C.POINTER(C.c_float)


class IndexDesc(C.Structure):
    _fields_ = [
        ("dim", C.c_uint32), ("nbits", C.c_uint32),
        ("num_centroids", C.c_uint64), ("num_passages", C.c_uint64), ("num_embeddings", C.c_uint64),
        ("centroids", f32p), ("codes", u32p), ("residuals", u8p), ("doclens", u32p),
        ("ivf_offsets", u64p), ("ivf_postings", u32p),
        ("bucket_cutoffs", f32p), ("bucket_weights", f32p),
    ]


class Params(C.Structure):
    _fields_ = [("k", C.c_uint64), ("nprobe", C.c_uint64), ("t_cs", C.c_float),
                ("ndocs", C.c_uint64), ("disable_filter", C.c_int32)]


class Trace(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "stage1_candidates", "stage2_out", "stage3_out", "final_out", "centroid_matmul_count",
        "stage2_rows_gathered", "stage3_rows_gathered", "decompressed_passages")] + \
        [(n, C.c_double) for n in (
            "candidate_generation_ms", "stage2_ms", "stage3_ms", "lookup_ms", "decompression_ms",
            "scoring_ms", "total_ms")] + [("decompressed_tokens", C.c_uint64)]


class EncodeDesc(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("nbits", C.c_uint32), ("num_centroids", C.c_uint64),
                ("num_passages", C.c_uint64), ("num_embeddings", C.c_uint64), ("embeddings", C.c_void_p),
                ("doclens", C.c_void_p), ("centroids", C.c_void_p), ("bucket_cutoffs", C.c_void_p)]


class SynthDesc(C.Structure):
    _fields_ = [("num_passages", C.c_uint64), ("num_centroids", C.c_uint64), ("pid_base", C.c_uint64),
                ("seed", C.c_uint64), ("dim", C.c_uint32), ("nbits", C.c_uint32), ("mean_len", C.c_uint32),
                ("spread", C.c_uint32), ("repeat", C.c_double)]


class BuildDesc(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("nbits", C.c_uint32), ("num_passages", C.c_uint64),
                ("num_embeddings", C.c_uint64), ("embeddings", C.c_void_p), ("doclens", C.c_void_p),
                ("num_centroids", C.c_uint64), ("kmeans_iters", C.c_uint64), ("rng_seed", C.c_uint64)]


class SearcherConfig(C.Structure):
    _fields_ = [("score_mode", C.c_int32), ("record_times", C.c_int32),
                ("use_graphs", C.c_int32), ("batch_engine", C.c_int32)]


# name -> (restype, argtypes); every symbol declared in include/plaid.h
SIGNATURES = {
    "plaid_last_error": (C.c_char_p, []),
    "plaid_status_name": (C.c_char_p, [C.c_int]),
    "plaid_abi_version": (C.c_int, []),
    "plaid_validate_query": (C.c_int, [f32p, C.c_uint64, C.c_uint64, C.c_uint64]),
    "plaid_validate_params": (C.c_int, [C.POINTER(Params), C.c_uint64]),
    "plaid_default_params_for_k": (None, [C.c_uint64, C.POINTER(Params)]),
    "plaid_stage3_width": (C.c_uint64, [C.POINTER(Params)]),
    "plaid_index_from_host": (C.c_int, [C.POINTER(IndexDesc), C.c_int, C.c_int, C.POINTER(C.c_void_p)]),
    "plaid_index_from_host_at": (C.c_int, [C.POINTER(IndexDesc), C.c_uint64, C.c_int, C.POINTER(C.c_void_p)]),
    "plaid_index_from_host_shard":(C.c_int, [C.POINTER(IndexDesc), C.c_uint64, C.c_uint64, C.c_int,
                                              C.POINTER(C.c_void_p)]),
    "plaid_index_validate": (C.c_int, [C.c_void_p]),
    "plaid_index_close": (None, [C.c_void_p]),
    "plaid_index_info": (None, [C.c_void_p, u64p]),
    "plaid_searcher_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(SearcherConfig), C.POINTER(C.c_void_p)]),
    "plaid_searcher_destroy": (None, [C.c_void_p]),
    # hot host path: array arguments as raw addresses (a ctypes POINTER per
    # argument costs several microseconds per call)
    "plaid_search": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(Params), C.c_void_p,
                               C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(Trace)]),
    "plaid_search_batch": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Params),
                                     u32p, f32p, u64p, C.POINTER(Trace)]),
    "plaid_search_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.POINTER(Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    "plaid_encode": (C.c_int, [C.POINTER(EncodeDesc), C.c_int, u32p, u8p, u64p, u32p, C.c_uint64, u64p]),
    "plaid_index_save": (C.c_int, [C.POINTER(IndexDesc), C.c_char_p, C.c_uint64]),
    "plaid_index_open": (C.c_int, [C.c_char_p, C.c_int, C.c_uint32, C.POINTER(C.c_void_p)]),
    "plaid_checksum": (C.c_uint64, [C.c_void_p, C.c_uint64]),
    "plaid_measure_read_gbs": (C.c_int, [C.c_int, C.c_uint64, C.c_int, C.POINTER(C.c_double)]),
    "plaid_batch_create": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(SearcherConfig), C.c_uint32,
                                     C.POINTER(C.c_void_p)]),
    "plaid_batch_destroy": (None, [C.c_void_p]),
    "plaid_batch_search": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Params),
                                     u32p, f32p, u64p]),
    "plaid_batch_search_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_uint64,
                                            C.POINTER(Params), C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64]),
    "plaid_batch_sync": (C.c_int, [C.c_void_p]),
    "plaid_batch_last_launches": (C.c_uint64, [C.c_void_p]),
    "plaid_batch_counters": (C.c_int, [C.c_void_p, u64p, C.c_uint64]),
    "plaid_batch_last_was_wave": (C.c_int, [C.c_void_p]),
    "plaid_batch_wave_slots": (C.c_uint32, [C.c_void_p]),
    "plaid_batch_wave_scores": (C.c_int, [C.c_void_p, C.c_uint64, f32p]),
    "plaid_shard_phase1_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(Params),
                                            C.c_void_p, C.c_uint64, C.c_uint64]),
    "plaid_shard_phase2_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64,
                                            C.c_uint64]),
    "plaid_shard_phase3_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_uint64]),
    "plaid_searcher_trace_counters_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "plaid_searcher_sync": (C.c_int, [C.c_void_p]),
    "plaid_searcher_last_launches": (C.c_uint64, [C.c_void_p]),
    "plaid_searcher_phase_ms": (C.c_int, [C.c_void_p, C.POINTER(C.c_double)]),
    "plaid_merge_topk": (C.c_int, [C.c_void_p, u32p, f32p, u64p, C.c_uint64, C.c_uint64, C.c_uint64,
                                   u32p, f32p, u64p]),
    "plaid_merge_topk_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.c_uint64]),
    "plaid_merge_topk_rows_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p,
                                               C.c_void_p, C.c_void_p, C.c_uint64]),
    "plaid_compute_centroid_scores": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_uint64, f32p, f32p]),
    "plaid_generate_candidates": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_uint64, u32p, u64p]),
    "plaid_prune_centroids": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_float, u8p]),
    "plaid_centroid_interaction": (C.c_int, [C.c_void_p, f32p, C.c_uint64, u32p, C.c_uint64, u8p, f32p, u64p]),
    "plaid_select_top": (C.c_int, [C.c_void_p, u32p, f32p, C.c_uint64, C.c_uint64, u32p, f32p, u64p]),
    "plaid_rank_final": (C.c_int, [C.c_void_p, f32p, C.c_uint64, u32p, C.c_uint64, C.c_uint64, u32p, f32p,
                                   u64p]),
    "plaid_reconstruct": (C.c_int, [C.c_void_p, u32p, C.c_uint64, u8p, f32p]),
    "plaid_lut_build": (C.c_int, [C.c_uint32, u8p]),
    "plaid_unpack_via_lut": (C.c_int, [C.c_void_p, u8p, C.c_uint64, C.c_uint32, u8p]),
    "plaid_pack_residual": (C.c_int, [u8p, C.c_uint64, C.c_uint32, u8p]),
    "plaid_maxsim_packed": (C.c_int, [C.c_void_p, f32p, C.c_uint64, u64p, C.c_uint64, f32p]),
    "plaid_maxsim_embeddings": (C.c_int, [C.c_void_p, f32p, C.c_uint64, C.c_uint64, f32p, u64p, C.c_uint64,
                                          f32p]),
    "plaid_merge_topk_batch_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64,
                                                C.c_uint64, C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_uint64]),
    "plaid_sharded_create": (C.c_int, [C.POINTER(C.c_void_p), C.c_uint32, C.POINTER(SearcherConfig), C.c_int32,
                                       C.POINTER(C.c_void_p)]),
    "plaid_sharded_destroy": (None, [C.c_void_p]),
    "plaid_sharded_search": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint64, C.POINTER(Params),
                                       C.c_void_p, C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(Trace)]),
    "plaid_sharded_last_launches": (C.c_uint64, [C.c_void_p]),
    "plaid_index_synth": (C.c_int, [C.POINTER(SynthDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "plaid_index_synth_queries": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_double, C.c_uint64,
                                            C.c_void_p]),
    "plaid_index_export": (C.c_int, [C.c_void_p] + [C.c_void_p] * 8),
    "plaid_build_index": (C.c_int, [C.POINTER(BuildDesc), C.c_int, C.c_void_p, C.c_uint64, C.POINTER(C.c_uint64),
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                    C.c_uint64, C.POINTER(C.c_uint64)]),
    # test knobs (not part of include/plaid.h)
    "plaid_debug_set_tf32_grid": (C.c_uint32, [C.c_uint32]),
    "plaid_debug_set_launch_cap": (C.c_longlong, [C.c_longlong]),
    "plaid_debug_wave_trace": (C.c_int, [C.c_void_p, u64p, C.c_uint64]),
    "plaid_debug_rs2_trace": (C.c_int, [C.c_int, C.c_void_p]),
}

_lib = None


def lib_path() -> Path:
    # PLAID_LIB: an alternative build of the same library (A/B timing runs)
    return Path(os.environ["PLAID_LIB"]) if os.environ.get("PLAID_LIB") else _LIB_DIR / "libplaid.so"


def load() -> C.CDLL:
    """Load libplaid.so (build it with __graft_entry__.build() first)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise RuntimeError(f"{path} is missing: the CUDA engine is not built "
                           "(run `python -c 'import __graft_entry__ as g; g.build()'`); "
                           "there is no CPU fallback")
    lib = C.CDLL(str(path))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def ptr(a, ctype):
    """ctypes pointer to a numpy array's data (None for None)."""
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))

"""Python mirror of the reference searcher's interface (namespace `lir`,
/root/reference/proj/include/lir/*.hpp) over the C ABI of libplaid.so.

Names, argument meaning and error behaviour follow the reference:
`search` (pipeline.hpp:86-87), the per-stage functions (pipeline.hpp:55-90),
the codec (residual_codec.hpp) and MaxSim kernels (maxsim.hpp).  Errors raise
`PlaidError` whose `.code` is the lir::ErrorCode (error.hpp:8-26).  Every call
runs on the GPU; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import struct
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native as N
from .hostindex import HostIndex


class ErrorCode(enum.IntEnum):  # error.hpp:8-26 (+1 on the wire)
    DimensionMismatch = 0
    NotNormalized = 1
    TooFewPoints = 2
    PackingUnsupported = 3
    EmptyCorpus = 4
    IndexOutOfRange = 5
    LengthNotPackable = 6
    EmptyPassageRange = 7
    InvalidParams = 8
    ChecksumMismatch = 9
    UnsupportedVersion = 10
    InvariantViolation = 11
    HeaderMismatch = 12
    NormalizationError = 13
    LengthMismatch = 14
    UnknownQueryId = 15
    IoError = 16
    CudaError = 99
    NcclError = 100
    Unsupported = 101
    OutOfMemory = 102


class PlaidError(RuntimeError):
    """lir::Error (error.hpp:51-61): carries an ErrorCode."""

    def __init__(self, code: ErrorCode, message: str):
        super().__init__(f"{code.name}: {message}")
        self.code = code


def _check(status: int) -> None:
    if status != 0:
        msg = N.load().plaid_last_error().decode(errors="replace")
        raise PlaidError(ErrorCode(status - 1), msg)


class ScoreMode(enum.IntEnum):
    TENSOR = 0
    EXACT = 1


@dataclass
class SearchParams:  # types.hpp:79-84
    k: int = 10
    nprobe: int = 1
    t_cs: float = 0.5
    ndocs: int = 256

    def _c(self, disable_filter: bool = False) -> N.Params:
        return N.Params(int(self.k), int(self.nprobe), float(self.t_cs), int(self.ndocs), int(bool(disable_filter)))


@dataclass
class SearchOptions:  # pipeline.hpp:45-48
    threads: int = 0             # accepted for interface parity; the grid size is internal
    disable_filter: bool = False


@dataclass
class CandidateSet:  # types.hpp:93-99
    passage_ids: np.ndarray
    scores: Optional[np.ndarray] = None

    def __len__(self) -> int:
        return int(self.passage_ids.shape[0])


@dataclass
class StageTrace:  # pipeline.hpp:23-43
    stage1_candidates: int = 0
    stage2_out: int = 0
    stage3_out: int = 0
    final_out: int = 0
    candidate_generation_ms: float = 0.0
    stage2_ms: float = 0.0
    stage3_ms: float = 0.0
    lookup_ms: float = 0.0
    decompression_ms: float = 0.0
    scoring_ms: float = 0.0
    total_ms: float = 0.0
    centroid_matmul_count: int = 0
    stage2_rows_gathered: int = 0
    stage3_rows_gathered: int = 0
    decompressed_passages: int = 0
    decompressed_tokens: int = 0  # stage-4 tokens (engine extra, not a lir counter)

    @classmethod
    def _from_c(cls, t: N.Trace) -> "StageTrace":
        # one struct.unpack of the C struct, reordered into this class's fields
        v = _TRACE_STRUCT.unpack(bytes(t))
        return cls(*[v[i] for i in _TRACE_PERM])

    def filtering_ms(self) -> float:
        return self.stage2_ms + self.stage3_ms

    def counters(self) -> dict:
        return {k: getattr(self, k) for k in (
            "stage1_candidates", "stage2_out", "stage3_out", "final_out", "centroid_matmul_count",
            "stage2_rows_gathered", "stage3_rows_gathered", "decompressed_passages")}


def _addr(a: np.ndarray) -> int:
    """Data address of a contiguous array (the buffer protocol is ~2x faster
    than __array_interface__ on the search path; read-only arrays fall back)."""
    try:
        return C.addressof(C.c_char.from_buffer(a))
    except (TypeError, ValueError):
        return a.ctypes.data


_TRACE_STRUCT = struct.Struct("<8Q7dQ")  # N.Trace's layout
assert _TRACE_STRUCT.size == C.sizeof(N.Trace)
_TRACE_PERM = [[f for f, _ in N.Trace._fields_].index(g.name) for g in dataclasses.fields(StageTrace)]


@dataclass
class SearchResult:  # pipeline.hpp:50-53
    topk: CandidateSet
    trace: StageTrace = field(default_factory=StageTrace)


def default_params_for_k(k: int) -> SearchParams:  # types.cpp:74-86
    p = N.Params()
    N.load().plaid_default_params_for_k(int(k), C.byref(p))
    return SearchParams(int(p.k), int(p.nprobe), float(p.t_cs), int(p.ndocs))


def stage3_width(params: SearchParams) -> int:  # pipeline.cpp:227-230
    return int(N.load().plaid_stage3_width(C.byref(params._c())))


def validate_params(params: SearchParams, num_centroids: int) -> None:  # types.cpp:88-99
    _check(N.load().plaid_validate_params(C.byref(params._c()), int(num_centroids)))


def validate_query(q: np.ndarray, index_dim: int) -> None:  # types.cpp:61-72
    q = np.ascontiguousarray(q, dtype=np.float32)
    rows, dim = (q.shape if q.ndim == 2 else (0, q.shape[-1] if q.ndim else 0))
    _check(N.load().plaid_validate_query(N.ptr(q, C.c_float), rows, dim, int(index_dim)))


def lut_build(nbits: int) -> np.ndarray:  # residual_codec.cpp:42-59
    if nbits not in (1, 2, 4):
        raise PlaidError(ErrorCode.PackingUnsupported, f"nbits {nbits} not in {{1,2,4}}")
    t = np.zeros(256 * (8 // nbits), dtype=np.uint8)
    _check(N.load().plaid_lut_build(nbits, N.ptr(t, C.c_uint8)))
    return t.reshape(256, 8 // nbits)


def pack_residual(bucket_indices: np.ndarray, nbits: int) -> np.ndarray:  # residual_codec.cpp:61-84
    idx = np.ascontiguousarray(bucket_indices, dtype=np.uint8)
    if nbits not in (1, 2, 4):
        raise PlaidError(ErrorCode.PackingUnsupported, f"nbits {nbits} not in {{1,2,4}}")
    out = np.zeros(max(1, idx.size * nbits // 8), dtype=np.uint8)
    _check(N.load().plaid_pack_residual(N.ptr(idx, C.c_uint8), idx.size, nbits, N.ptr(out, C.c_uint8)))
    return out[: idx.size * nbits // 8]


def _desc(h: HostIndex) -> N.IndexDesc:
    return N.IndexDesc(h.dim, h.nbits, h.num_centroids, h.num_passages, h.num_embeddings,
                       N.ptr(h.centroids, C.c_float), N.ptr(h.codes, C.c_uint32),
                       N.ptr(h.residuals, C.c_uint8), N.ptr(h.doclens, C.c_uint32),
                       N.ptr(h.ivf_offsets, C.c_uint64), N.ptr(h.ivf_postings, C.c_uint32),
                       N.ptr(h.bucket_cutoffs, C.c_float), N.ptr(h.bucket_weights, C.c_float))


def encode_corpus(embeddings: np.ndarray, doclens: np.ndarray, centroids: np.ndarray, bucket_cutoffs: np.ndarray,
                  bucket_weights: np.ndarray, nbits: int, device: int = 0) -> HostIndex:
    """The encode half of lir::build_index on the GPU (indexer.cpp:197-282):
    codes (exact assign_codes), packed residuals and the IVF for trained
    centroids + quantizer; returns the HostIndex (bit-identical to the
    reference's)."""
    emb = np.ascontiguousarray(embeddings, dtype=np.float32)
    dl = np.ascontiguousarray(doclens, dtype=np.uint32)
    cents = np.ascontiguousarray(centroids, dtype=np.float32)
    cut = np.ascontiguousarray(bucket_cutoffs, dtype=np.float32)
    T, dim = emb.shape
    K = cents.shape[0]
    d = N.EncodeDesc(dim, nbits, K, dl.size, T, emb.ctypes.data, dl.ctypes.data, cents.ctypes.data, cut.ctypes.data)
    codes = np.zeros(max(T, 1), dtype=np.uint32)
    res = np.zeros(max(T * nbits * dim // 8, 1), dtype=np.uint8)
    ivo = np.zeros(K + 1, dtype=np.uint64)
    post = np.zeros(max(T, 1), dtype=np.uint32)
    n = C.c_uint64()
    _check(N.load().plaid_encode(C.byref(d), device, N.ptr(codes, C.c_uint32), N.ptr(res, C.c_uint8),
                                 N.ptr(ivo, C.c_uint64), N.ptr(post, C.c_uint32), post.size, C.byref(n)))
    return HostIndex(dim, nbits, cents, codes[:T], res[: T * nbits * dim // 8], dl, ivo, post[: n.value], cut,
                     np.ascontiguousarray(bucket_weights, dtype=np.float32))


def build_index(embeddings: np.ndarray, doclens: np.ndarray, nbits: int = 2, num_centroids: int = 0,
                iters: int = 20, seed: int = 42, device: int = 0) -> HostIndex:
    """lir::build_index (indexer.cpp:197-282) on the GPU: k-means, quantizer,
    codes, residuals and IVF, bit-identical to the reference for the same
    corpus, IndexConfig (nbits, num_centroids 0 = auto, kmeans_iters,
    rng_seed) — plaid_build_index."""
    x = np.ascontiguousarray(embeddings, dtype=np.float32)
    dl = np.ascontiguousarray(doclens, dtype=np.uint32)
    T, dim = x.shape
    k = int(num_centroids) if num_centroids else (min(1 << int(np.ceil(np.log2(T) / 2.0)), T) if T else 1)
    cents = np.empty((max(k, 1), dim), np.float32)
    nb = 1 << nbits
    cut = np.zeros(16, np.float32)
    w = np.zeros(16, np.float32)
    codes = np.empty(max(T, 1), np.uint32)
    res = np.empty(max(T * nbits * dim // 8, 1), np.uint8)
    ivo = np.empty(k + 1, np.uint64)
    post = np.empty(max(T, 1), np.uint32)
    kk, P = C.c_uint64(), C.c_uint64()
    d = N.BuildDesc(dim, nbits, dl.size, T, x.ctypes.data, dl.ctypes.data, int(num_centroids), int(iters), int(seed))
    _check(N.load().plaid_build_index(C.byref(d), device, cents.ctypes.data, k, C.byref(kk), cut.ctypes.data,
                                      w.ctypes.data, codes.ctypes.data, res.ctypes.data, ivo.ctypes.data,
                                      post.ctypes.data, post.size, C.byref(P)))
    return HostIndex(dim, nbits, cents[: kk.value], codes[:T], res[: T * nbits * dim // 8], dl, ivo[: kk.value + 1],
                     post[: P.value], cut[: nb - 1], w[:nb])


def save_index(h: HostIndex, path: str, rng_seed: int = 0) -> None:
    """Write `h` in the on-disk format (FORMAT.md; SPEC.md storage module)."""
    d = _desc(h)
    _check(N.load().plaid_index_save(C.byref(d), str(path).encode(), int(rng_seed)))


def checksum(buf: np.ndarray) -> int:
    """FORMAT.md digest of a host array (the manifest's per-file checksum)."""
    b = np.ascontiguousarray(buf)
    return int(N.load().plaid_checksum(b.ctypes.data_as(C.c_void_p), b.nbytes))


class DeviceIndex:
    """The compressed index resident in HBM (index.hpp:60-85).  Immutable and
    shareable between searchers (index.hpp:57-59)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        info = (C.c_uint64 * 8)()
        N.load().plaid_index_info(self._h, info)
        (self.dim, self.nbits, self.num_centroids, self.num_passages, self.num_embeddings,
         self.num_postings, self.pid_base, self.device_bytes) = (int(x) for x in info)

    @classmethod
    def from_host(cls, h: HostIndex, device: int = 0, validate: bool = False) -> "DeviceIndex":
        out = C.c_void_p()
        d = _desc(h)
        _check(N.load().plaid_index_from_host(C.byref(d), device, int(validate), C.byref(out)))
        return cls(out.value)

    @classmethod
    def from_host_at(cls, h: HostIndex, pid_base: int, device: int = 0) -> "DeviceIndex":
        """`h` is already the shard [pid_base, pid_base + N) with local ids."""
        out = C.c_void_p()
        d = _desc(h)
        _check(N.load().plaid_index_from_host_at(C.byref(d), int(pid_base), device, C.byref(out)))
        return cls(out.value)

    @classmethod
    def shard(cls, h: HostIndex, pid_begin: int, pid_end: int, device: int = 0) -> "DeviceIndex":
        out = C.c_void_p()
        d = _desc(h)
        _check(N.load().plaid_index_from_host_shard(C.byref(d), pid_begin, pid_end, device, C.byref(out)))
        return cls(out.value)

    @classmethod
    def open(cls, path: str, device: int = 0, validate: bool = False, checksums: bool = True) -> "DeviceIndex":
        """Load an on-disk index (FORMAT.md): mmap, one upload to HBM, every
        file checksum verified on the GPU over the uploaded arrays."""
        out = C.c_void_p()
        flags = (1 if validate else 0) | (0 if checksums else 2)
        _check(N.load().plaid_index_open(str(path).encode(), device, flags, C.byref(out)))
        return cls(out.value)

    @classmethod
    def synth(cls, num_passages: int, num_centroids: int, dim: int = 128, nbits: int = 2, mean_len: int = 64,
              spread: int = 16, repeat: float = 0.28, seed: int = 0, pid_base: int = 0,
              device: int = 0) -> "DeviceIndex":
        """The synthetic corpus of generate_index (same arguments, same integer
        arrays) generated directly in HBM: passages [pid_base, pid_base + N)
        with a local IVF and global ids in results (plaid_index_synth)."""
        d = N.SynthDesc(int(num_passages), int(num_centroids), int(pid_base), int(seed), int(dim), int(nbits),
                        int(mean_len), int(spread), float(repeat))
        out = C.c_void_p()
        _check(N.load().plaid_index_synth(C.byref(d), device, C.byref(out)))
        return cls(out.value)

    def synth_queries(self, num_queries: int, qlen: int = 32, noise: float = 0.03, seed: int = 1234) -> np.ndarray:
        """generate_queries' recipe on the device-resident index."""
        out = np.empty((num_queries, qlen, self.dim), dtype=np.float32)
        _check(N.load().plaid_index_synth_queries(self._h, num_queries, qlen, float(noise), seed, out.ctypes.data))
        return out

    def to_host(self) -> HostIndex:
        """Download the index arrays (plaid_index_export)."""
        nb = 1 << self.nbits
        a = dict(centroids=np.empty((self.num_centroids, self.dim), np.float32),
                 codes=np.empty(self.num_embeddings, np.uint32),
                 residuals=np.empty(self.num_embeddings * self.nbits * self.dim // 8, np.uint8),
                 doclens=np.empty(self.num_passages, np.uint32),
                 ivf_offsets=np.empty(self.num_centroids + 1, np.uint64),
                 ivf_postings=np.empty(max(self.num_postings, 1), np.uint32),
                 bucket_cutoffs=np.empty(max(nb - 1, 1), np.float32), bucket_weights=np.empty(nb, np.float32))
        order = ("centroids", "codes", "residuals", "doclens", "ivf_offsets", "ivf_postings", "bucket_cutoffs",
                 "bucket_weights")
        _check(N.load().plaid_index_export(self._h, *[a[k].ctypes.data for k in order]))
        return HostIndex(self.dim, self.nbits, a["centroids"], a["codes"], a["residuals"], a["doclens"],
                         a["ivf_offsets"], a["ivf_postings"][: self.num_postings], a["bucket_cutoffs"][: nb - 1],
                         a["bucket_weights"])

    def validate(self) -> None:  # index.cpp:12-84
        _check(N.load().plaid_index_validate(self._h))

    def close(self) -> None:
        if self._h:
            N.load().plaid_index_close(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Searcher:
    """One CUDA stream + device scratch; use one per host thread."""

    def __init__(self, index: Optional[DeviceIndex] = None, device: int = 0,
                 score_mode: ScoreMode = ScoreMode.EXACT, record_times: bool = True,
                 use_graphs: bool = False):
        self.index = index
        cfg = N.SearcherConfig(int(score_mode), int(record_times), int(use_graphs), 0)
        out = C.c_void_p()
        _check(N.load().plaid_searcher_create(index._h if index else None, device, C.byref(cfg), C.byref(out)))
        self._h = out
        self._lib = N.load()
        self._call = None  # search(): cached C arguments

    def close(self) -> None:
        if self._h:
            N.load().plaid_searcher_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- lir::search
    def search(self, q: np.ndarray, params: SearchParams, options: SearchOptions = SearchOptions()) -> SearchResult:
        q = np.ascontiguousarray(q, dtype=np.float32)
        if q.ndim != 2:
            raise PlaidError(ErrorCode.DimensionMismatch, "query must be rows x dim")
        # the C arguments of the last (params, options) are kept: output
        # buffers, their addresses and the byref'd structs (a Searcher serves
        # one host thread)
        key = (params.k, params.nprobe, params.t_cs, params.ndocs, options.disable_filter)
        c = self._call
        if c is None or c[0] != key:
            k = max(int(params.k), 1)
            ids, sc = np.empty(k, dtype=np.uint32), np.empty(k, dtype=np.float32)
            cp, n, tr = params._c(options.disable_filter), C.c_uint64(), N.Trace()
            c = self._call = (key, ids, sc, n, tr, C.byref(cp), ids.ctypes.data, sc.ctypes.data, C.byref(n),
                              C.byref(tr), cp)
        _, ids, sc, n, tr, cp_ref, ia, sa, n_ref, tr_ref, _cp = c
        _check(self._lib.plaid_search(self._h, _addr(q), q.shape[0], q.shape[1], cp_ref, ia, sa, n_ref, tr_ref))
        m = n.value
        return SearchResult(CandidateSet(ids[:m].copy(), sc[:m].copy()), StageTrace._from_c(tr))

    def search_batch(self, q: np.ndarray, params: SearchParams, options: SearchOptions = SearchOptions()):
        q = np.ascontiguousarray(q, dtype=np.float32)
        nq, rows, dim = q.shape
        k = int(params.k)
        ids = np.zeros((nq, k), dtype=np.uint32)
        sc = np.zeros((nq, k), dtype=np.float32)
        n = np.zeros(nq, dtype=np.uint64)
        p = params._c(options.disable_filter)
        _check(N.load().plaid_search_batch(self._h, N.ptr(q, C.c_float), nq, rows, dim, C.byref(p),
                                           N.ptr(ids, C.c_uint32), N.ptr(sc, C.c_float), N.ptr(n, C.c_uint64),
                                           None))
        return ids, sc, n

    def search_device(self, d_q: int, nq: int, rows: int, dim: int, params: SearchParams,
                      d_pids: int, d_scores: int, d_n: int, stream: int = 0,
                      options: SearchOptions = SearchOptions()) -> None:
        p = params._c(options.disable_filter)
        _check(N.load().plaid_search_device(self._h, d_q, nq, rows, dim, C.byref(p), d_pids, d_scores, d_n,
                                            stream))

    def merge_topk_device(self, d_pids: int, d_scores: int, d_counts: int, shards: int, stride: int, k: int,
                          d_out_pids: int, d_out_scores: int, d_out_n: int, stream: int = 0) -> None:
        """Device-side final select over G gathered shard lists."""
        _check(N.load().plaid_merge_topk_device(self._h, d_pids, d_scores, d_counts, shards, stride, k,
                                                d_out_pids, d_out_scores, d_out_n, stream))

    # ---- global-exact passage sharding (include/plaid.h)
    def shard_phase1(self, d_q: int, rows: int, dim: int, params: SearchParams, d_x2: int, stride2: int,
                     stream: int = 0, options: SearchOptions = SearchOptions()) -> None:
        p = params._c(options.disable_filter)
        _check(N.load().plaid_shard_phase1_device(self._h, d_q, rows, dim, C.byref(p), d_x2, stride2, stream))

    def shard_phase2(self, d_g2: int, shards: int, d_x3: int, stride3: int, stream: int = 0) -> None:
        _check(N.load().plaid_shard_phase2_device(self._h, d_g2, shards, d_x3, stride3, stream))

    def shard_phase3(self, d_g3: int, shards: int, d_pids: int, d_scores: int, d_n: int, stream: int = 0) -> None:
        _check(N.load().plaid_shard_phase3_device(self._h, d_g3, shards, d_pids, d_scores, d_n, stream))

    def trace_counters_device(self, d_out: int, stream: int = 0) -> None:
        _check(N.load().plaid_searcher_trace_counters_device(self._h, d_out, stream))

    def merge_topk_rows_device(self, d_rows: int, shards: int, k: int, d_out_pids: int, d_out_scores: int,
                               d_out_n: int, stream: int = 0) -> None:
        """Merge packed per-shard rows [k pids | k scores | u64 count] (one all-gather per query)."""
        _check(N.load().plaid_merge_topk_rows_device(self._h, d_rows, shards, k, d_out_pids, d_out_scores,
                                                     d_out_n, stream))

    def sync(self) -> None:
        _check(N.load().plaid_searcher_sync(self._h))

    def last_launches(self) -> int:
        return int(N.load().plaid_searcher_last_launches(self._h))

    PHASES = ("scores", "candidates", "stage2_interaction", "stage2_select", "stage3", "stage4_rank",
              "final_select")

    def phase_ms(self) -> dict:
        """CUDA-event phase durations of the last enqueued query (record_times)."""
        out = (C.c_double * 7)()
        _check(N.load().plaid_searcher_phase_ms(self._h, out))
        return dict(zip(self.PHASES, list(out)))

    # ---- per-stage functions (pipeline.hpp:55-90)
    def compute_centroid_scores(self, q: np.ndarray):
        q = np.ascontiguousarray(q, dtype=np.float32)
        K = self.index.num_centroids
        S = np.zeros((K, q.shape[0]), dtype=np.float32)
        mx = np.zeros(K, dtype=np.float32)
        _check(N.load().plaid_compute_centroid_scores(self._h, N.ptr(q, C.c_float), q.shape[0], q.shape[1],
                                                      N.ptr(S, C.c_float), N.ptr(mx, C.c_float)))
        return S, mx

    def generate_candidates(self, scores: np.ndarray, nprobe: int) -> np.ndarray:
        S = np.ascontiguousarray(scores, dtype=np.float32)
        out = np.zeros(max(self.index.num_passages, 1), dtype=np.uint32)
        n = C.c_uint64()
        _check(N.load().plaid_generate_candidates(self._h, N.ptr(S, C.c_float), S.shape[1], int(nprobe),
                                                  N.ptr(out, C.c_uint32), C.byref(n)))
        return out[: n.value].copy()

    def prune_centroids(self, row_max: np.ndarray, t_cs: float) -> np.ndarray:
        mx = np.ascontiguousarray(row_max, dtype=np.float32)
        keep = np.zeros(mx.size, dtype=np.uint8)
        _check(N.load().plaid_prune_centroids(self._h, N.ptr(mx, C.c_float), mx.size, float(t_cs),
                                              N.ptr(keep, C.c_uint8)))
        return keep

    def centroid_interaction(self, candidates: np.ndarray, scores: np.ndarray, mask: Optional[np.ndarray]):
        cand = np.ascontiguousarray(candidates, dtype=np.uint32)
        S = np.ascontiguousarray(scores, dtype=np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.zeros(max(cand.size, 1), dtype=np.float32)
        rows = C.c_uint64()
        _check(N.load().plaid_centroid_interaction(self._h, N.ptr(S, C.c_float), S.shape[1],
                                                   N.ptr(cand, C.c_uint32), cand.size, N.ptr(m, C.c_uint8),
                                                   N.ptr(out, C.c_float), C.byref(rows)))
        return out[: cand.size].copy(), int(rows.value)

    def select_top(self, ids: np.ndarray, scores: np.ndarray, n: int):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        sc = np.ascontiguousarray(scores, dtype=np.float32)
        m = max(min(int(n), ids.size), 1)
        oi = np.zeros(m, dtype=np.uint32)
        os_ = np.zeros(m, dtype=np.float32)
        cnt = C.c_uint64()
        _check(N.load().plaid_select_top(self._h, N.ptr(ids, C.c_uint32), N.ptr(sc, C.c_float), ids.size, int(n),
                                         N.ptr(oi, C.c_uint32), N.ptr(os_, C.c_float), C.byref(cnt)))
        return oi[: cnt.value].copy(), os_[: cnt.value].copy()

    def rank_final(self, candidates: np.ndarray, q: np.ndarray, k: int):
        cand = np.ascontiguousarray(candidates, dtype=np.uint32)
        q = np.ascontiguousarray(q, dtype=np.float32)
        m = max(min(int(k), cand.size), 1)
        oi = np.zeros(m, dtype=np.uint32)
        os_ = np.zeros(m, dtype=np.float32)
        cnt = C.c_uint64()
        _check(N.load().plaid_rank_final(self._h, N.ptr(q, C.c_float), q.shape[0], N.ptr(cand, C.c_uint32),
                                         cand.size, int(k), N.ptr(oi, C.c_uint32), N.ptr(os_, C.c_float),
                                         C.byref(cnt)))
        return oi[: cnt.value].copy(), os_[: cnt.value].copy()

    # ---- codec / MaxSim
    def reconstruct(self, codes: np.ndarray, residuals: np.ndarray) -> np.ndarray:
        codes = np.ascontiguousarray(codes, dtype=np.uint32)
        res = np.ascontiguousarray(residuals, dtype=np.uint8).reshape(-1)
        out = np.zeros((codes.size, self.index.dim), dtype=np.float32)
        _check(N.load().plaid_reconstruct(self._h, N.ptr(codes, C.c_uint32), codes.size, N.ptr(res, C.c_uint8),
                                          N.ptr(out, C.c_float)))
        return out

    def unpack_via_lut(self, packed: np.ndarray, nbits: int) -> np.ndarray:
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        if nbits not in (1, 2, 4):
            raise PlaidError(ErrorCode.PackingUnsupported, f"nbits {nbits} not in {{1,2,4}}")
        out = np.zeros(max(pk.size * (8 // nbits), 1), dtype=np.uint8)
        _check(N.load().plaid_unpack_via_lut(self._h, N.ptr(pk, C.c_uint8), pk.size, nbits, N.ptr(out, C.c_uint8)))
        return out[: pk.size * (8 // nbits)]

    def maxsim_packed(self, scores: np.ndarray, offsets: np.ndarray) -> np.ndarray:
        S = np.ascontiguousarray(scores, dtype=np.float32)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        np_ = max(off.size - 1, 0)
        if off.size == 0:
            raise PlaidError(ErrorCode.InvalidParams, "offsets must start at 0")
        out = np.zeros(max(np_, 1), dtype=np.float32)
        nq = S.shape[1] if S.ndim == 2 else 0
        _check(N.load().plaid_maxsim_packed(self._h, N.ptr(S, C.c_float), nq, N.ptr(off, C.c_uint64), np_,
                                            N.ptr(out, C.c_float)))
        return out[:np_]

    def maxsim_embeddings(self, q: np.ndarray, emb: np.ndarray, offsets: np.ndarray) -> np.ndarray:
        q = np.ascontiguousarray(q, dtype=np.float32)
        e = np.ascontiguousarray(emb, dtype=np.float32)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        if off.size == 0:
            raise PlaidError(ErrorCode.InvalidParams, "offsets must start at 0")
        np_ = off.size - 1
        out = np.zeros(max(np_, 1), dtype=np.float32)
        _check(N.load().plaid_maxsim_embeddings(self._h, N.ptr(q, C.c_float), q.shape[0], q.shape[1],
                                                N.ptr(e, C.c_float), N.ptr(off, C.c_uint64), np_,
                                                N.ptr(out, C.c_float)))
        return out[:np_]

    def merge_topk_batch_device(self, d_pids: int, d_scores: int, d_counts: int, shards: int, batch: int, k: int,
                                d_out_pids: int, d_out_scores: int, d_out_n: int, stream: int = 0) -> None:
        """[shards][B][k] shard lists (+ counts [shards][B]) -> [B][k] global
        top-k per query, one kernel for the whole batch."""
        _check(N.load().plaid_merge_topk_batch_device(self._h, d_pids, d_scores, d_counts, shards, batch, k,
                                                      d_out_pids, d_out_scores, d_out_n, stream))

    def merge_topk(self, pids: np.ndarray, scores: np.ndarray, counts: np.ndarray, k: int):
        """Final select over G shard lists [G, stride]."""
        pids = np.ascontiguousarray(pids, dtype=np.uint32)
        sc = np.ascontiguousarray(scores, dtype=np.float32)
        cnt = np.ascontiguousarray(counts, dtype=np.uint64)
        G, stride = pids.shape
        oi = np.zeros(k, dtype=np.uint32)
        os_ = np.zeros(k, dtype=np.float32)
        n = C.c_uint64()
        _check(N.load().plaid_merge_topk(self._h, N.ptr(pids, C.c_uint32), N.ptr(sc, C.c_float),
                                         N.ptr(cnt, C.c_uint64), G, stride, k, N.ptr(oi, C.c_uint32),
                                         N.ptr(os_, C.c_float), C.byref(n)))
        return oi[: n.value].copy(), os_[: n.value].copy()


class MultiGpuSearcher:
    """lir::search over a passage-sharded index in ONE process
    (plaid_sharded_*, include/plaid.h): one searcher per shard on the
    shard's GPU, exchanges as on-device all-gathers over NVLink peer access,
    final select on shards[0]'s device.  mode "global-exact" equals the
    reference over the unsharded index; "shard-local" = reference per shard +
    top-k merge."""

    MODES = {"global-exact": 0, "shard-local": 1}

    def __init__(self, shards, score_mode: ScoreMode = ScoreMode.TENSOR, mode: str = "global-exact"):
        if mode not in self.MODES:
            raise ValueError(f"mode must be one of {tuple(self.MODES)}")
        self.shards = list(shards)
        arr = (C.c_void_p * len(self.shards))(*[s._h.value if isinstance(s._h, C.c_void_p) else s._h
                                                for s in self.shards])
        cfg = N.SearcherConfig(int(score_mode), 0, 0, 0)
        out = C.c_void_p()
        _check(N.load().plaid_sharded_create(arr, len(self.shards), C.byref(cfg), self.MODES[mode], C.byref(out)))
        self._h = out

    def close(self) -> None:
        if self._h:
            N.load().plaid_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, q: np.ndarray, params: SearchParams, options: SearchOptions = SearchOptions()) -> SearchResult:
        q = np.ascontiguousarray(q, dtype=np.float32)
        rows, dim = (q.shape if q.ndim == 2 else (0, 0))
        k = max(int(params.k), 1)
        ids = np.zeros(k, dtype=np.uint32)
        sc = np.zeros(k, dtype=np.float32)
        n = C.c_uint64()
        tr = N.Trace()
        p = params._c(options.disable_filter)
        _check(N.load().plaid_sharded_search(self._h, _addr(q), rows, dim, C.byref(p), _addr(ids), _addr(sc),
                                             C.byref(n), C.byref(tr)))
        m = n.value
        return SearchResult(CandidateSet(ids[:m].copy(), sc[:m].copy()), StageTrace._from_c(tr))

    def last_launches(self) -> int:
        return int(N.load().plaid_sharded_last_launches(self._h))


class BatchSearcher:
    """Throughput mode (BASELINE configs[2], batched queries).  Engine
    "auto": waves of queries — one S_cq pass per wave (four queries per pass
    over C in TENSOR mode) and one CTA per query for stages 1b-4 — whenever
    the shape allows, else (and with engine="lanes") `lanes` searchers with
    their own streams, query j on lane j mod lanes (include/plaid.h)."""

    def __init__(self, index: DeviceIndex, lanes: int = 8, device: int = 0,
                 score_mode: ScoreMode = ScoreMode.TENSOR, engine: str = "auto"):
        self.index = index
        if engine not in ("auto", "lanes"):
            raise PlaidError(ErrorCode.InvalidParams, f"unknown batch engine {engine!r}")
        cfg = N.SearcherConfig(int(score_mode), 0, 0, 1 if engine == "lanes" else 0)
        out = C.c_void_p()
        _check(N.load().plaid_batch_create(index._h, device, C.byref(cfg), int(lanes), C.byref(out)))
        self._h = out
        self.lanes = int(lanes)

    def close(self) -> None:
        if self._h:
            N.load().plaid_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def search(self, q: np.ndarray, params: SearchParams, options: SearchOptions = SearchOptions()):
        """q: [nq, rows, dim] float32 (host).  Returns a list of CandidateSet."""
        q = np.ascontiguousarray(q, dtype=np.float32)
        if q.ndim != 3:
            raise PlaidError(ErrorCode.DimensionMismatch, "queries must be nq x rows x dim")
        nq, rows, dim = q.shape
        k = max(int(params.k), 1)
        ids = np.zeros((nq, k), dtype=np.uint32)
        sc = np.zeros((nq, k), dtype=np.float32)
        n = np.zeros(nq, dtype=np.uint64)
        p = params._c(options.disable_filter)
        _check(N.load().plaid_batch_search(self._h, N.ptr(q, C.c_float), nq, rows, dim, C.byref(p),
                                           N.ptr(ids, C.c_uint32), N.ptr(sc, C.c_float), N.ptr(n, C.c_uint64)))
        # views into this call's fresh arrays (no per-query copies)
        return [CandidateSet(ids[j, :m], sc[j, :m]) for j, m in enumerate(n.tolist())]

    def search_device(self, d_q: int, nq: int, rows: int, dim: int, params: SearchParams, d_pids: int,
                      d_scores: int, d_n: int, stream: int = 0, options: SearchOptions = SearchOptions()) -> None:
        p = params._c(options.disable_filter)
        _check(N.load().plaid_batch_search_device(self._h, d_q, nq, rows, dim, C.byref(p), d_pids, d_scores, d_n,
                                                  stream))

    def sync(self) -> None:
        _check(N.load().plaid_batch_sync(self._h))

    def last_launches(self) -> int:
        return int(N.load().plaid_batch_last_launches(self._h))

    def last_was_wave(self) -> bool:
        return bool(N.load().plaid_batch_last_was_wave(self._h))

    def wave_slots(self) -> int:
        """Queries per wave of the wave engine (0 before its first batch)."""
        return int(N.load().plaid_batch_wave_slots(self._h))

    def wave_scores(self, j: int) -> np.ndarray:
        """Test hook: the [K, 32] S_cq table the last wave used for its j-th query."""
        out = np.zeros((self.index.num_centroids, 32), dtype=np.float32)
        _check(N.load().plaid_batch_wave_scores(self._h, j, N.ptr(out, C.c_float)))
        return out

    def counters(self, nq: int) -> np.ndarray:
        """[nq, 4] StageTrace counters (stage1_candidates, stage2_out,
        stage3_out, final_out) of the last batch (wave engine only)."""
        out = np.zeros((nq, 4), dtype=np.uint64)
        _check(N.load().plaid_batch_counters(self._h, N.ptr(out, C.c_uint64), nq))
        return out


def search(index: DeviceIndex, q: np.ndarray, params: SearchParams,
           options: SearchOptions = SearchOptions(), searcher: Optional[Searcher] = None) -> SearchResult:
    """lir::search (pipeline.hpp:86-87).  Creates a throwaway Searcher unless
    one is given; reuse a Searcher for repeated queries."""
    s = searcher or Searcher(index)
    return s.search(q, params, options)

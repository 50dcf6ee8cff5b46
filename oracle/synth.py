"""Benchmark-input generator on the checker side — TEST INFRASTRUCTURE ONLY.

oracle/synth_oracle.c restates SURVEY.md §8d's synthetic index recipe
independently of the product generator (paper_2205_09707_b200/csrc/synth), and
the IVF comes from the reference's own build_inverted_list
(indexer.cpp:149-195, oracle/_ref).  bench.py's `--impl reference` arm builds
its inputs here, so that arm maps no library of the product; tests/test_synth.py
checks the bytes equal the product generator's.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import HERE

_SO = HERE / "libsynth_oracle.so"
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not _SO.exists():
            raise FileNotFoundError(f"{_SO} not built (make -C oracle)")
        L = C.CDLL(str(_SO))
        vp, u64, u32, i32, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
        L.osyn_centroids.argtypes = [u64, u32, u64, vp, i32]
        L.osyn_doclens.argtypes = [u64, u64, u32, u32, u64, vp, i32]
        L.osyn_codes.argtypes = [vp, vp, u64, u64, u64, dbl, u64, vp, i32]
        L.osyn_residuals.argtypes = [vp, u64, u64, u64, u64, vp, i32]
        L.osyn_quantizer.argtypes = [u32, vp, vp]
        L.osyn_quantizer.restype = C.c_int
        L.osyn_queries.argtypes = [vp, u32, vp, vp, u32, vp, vp, vp, u64, u64, u32, dbl, u64, vp]
        _lib = L
    return _lib


@dataclass
class SynthIndex:
    """The persisted arrays of lir::CompressedIndex (index.hpp:60-85) + the
    derived passage offsets: the attribute surface the oracles read."""
    dim: int
    nbits: int
    centroids: np.ndarray
    codes: np.ndarray
    residuals: np.ndarray
    doclens: np.ndarray
    ivf_offsets: np.ndarray
    ivf_postings: np.ndarray
    bucket_cutoffs: np.ndarray
    bucket_weights: np.ndarray
    passage_offsets: np.ndarray

    @property
    def num_centroids(self) -> int:
        return int(self.centroids.shape[0])

    @property
    def num_passages(self) -> int:
        return int(self.doclens.size)

    @property
    def num_embeddings(self) -> int:
        return int(self.codes.size)

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.centroids, self.codes, self.residuals, self.doclens, self.ivf_offsets,
                                      self.ivf_postings, self.passage_offsets))


def _p(a):
    return a.ctypes.data


def generate_index(num_passages: int, num_centroids: int, dim: int = 128, nbits: int = 2, mean_len: int = 64,
                   spread: int = 16, repeat: float = 0.28, seed: int = 0, threads: int = 0, pid_base: int = 0,
                   ivf=None) -> SynthIndex:
    """Same arguments and bytes as paper_2205_09707_b200.generate_index.
    `ivf(codes, doclens, K) -> (offsets, postings)` builds the inverted list;
    default: the reference's build_inverted_list (oracle/_ref)."""
    L = _load()
    N, K = int(num_passages), int(num_centroids)
    cents = np.empty((K, dim), dtype=np.float32)
    L.osyn_centroids(K, dim, 11 + seed, _p(cents), threads)
    lo, hi = max(1, mean_len - spread), mean_len + spread
    doclens = np.empty(N, dtype=np.uint32)
    L.osyn_doclens(N, pid_base, lo, hi, 5 + seed, _p(doclens), threads)
    off = np.zeros(N + 1, dtype=np.uint64)
    np.cumsum(doclens, dtype=np.uint64, out=off[1:])
    T = int(off[-1])
    codes = np.empty(T, dtype=np.uint32)
    L.osyn_codes(_p(doclens), _p(off), N, pid_base, K, float(repeat), 99 + seed, _p(codes), threads)
    bpt = nbits * dim // 8
    res = np.empty(T * bpt, dtype=np.uint8)
    L.osyn_residuals(_p(off), N, pid_base, bpt, 7 + seed, _p(res), threads)
    if ivf is None:
        from . import get

        ivf = get("ref").build_inverted_list
    ivo, post = ivf(codes, doclens, K)
    nb = 1 << nbits
    cut = np.zeros(max(nb - 1, 1), dtype=np.float32)
    w = np.zeros(nb, dtype=np.float32)
    if L.osyn_quantizer(nbits, _p(cut), _p(w)) != 0:
        raise ValueError("nbits must be one of {1, 2, 4}")
    return SynthIndex(dim, nbits, cents, codes, res, doclens, np.ascontiguousarray(ivo, dtype=np.uint64),
                      np.ascontiguousarray(post, dtype=np.uint32), cut[: nb - 1], w, off)


def generate_queries(index, num_queries: int, qlen: int = 32, noise: float = 0.03, seed: int = 1234) -> np.ndarray:
    L = _load()
    out = np.empty((num_queries, qlen, index.dim), dtype=np.float32)
    L.osyn_queries(_p(index.centroids), index.dim, _p(index.codes), _p(index.residuals), index.nbits,
                   _p(index.bucket_weights), _p(index.doclens), _p(index.passage_offsets), index.num_passages,
                   num_queries, qlen, float(noise), seed, _p(out))
    return out

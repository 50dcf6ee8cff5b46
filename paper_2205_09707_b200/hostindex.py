"""Host-side index arrays (the persisted fields of lir::CompressedIndex,
reference include/lir/index.hpp:60-85) and the deterministic synthetic
generator that fills them (csrc/synth/synth.cpp).

The same HostIndex feeds the CUDA engine (`DeviceIndex.from_host`), the C
restatement in oracle/ and the compiled reference in oracle/_ref, which is
what makes bit-exact differential tests possible.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

_SYNTH = Path(__file__).resolve().parent / "_lib" / "libplaid_synth.so"
_synth = None


def _lib():
    global _synth
    if _synth is None:
        if not _SYNTH.exists():
            raise RuntimeError(f"{_SYNTH} missing; run __graft_entry__.build()")
        _synth = C.CDLL(str(_SYNTH))
        vp, u64, u32, i32, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_int, C.c_double
        _synth.synth_centroids.argtypes = [u64, u32, u64, vp, i32]
        _synth.synth_doclens.argtypes = [u64, u64, u32, u32, u64, vp, i32]
        _synth.synth_offsets.argtypes = [vp, u64, vp]
        _synth.synth_offsets.restype = u64
        _synth.synth_codes.argtypes = [vp, vp, u64, u64, u64, dbl, u64, vp, i32]
        _synth.synth_residuals.argtypes = [vp, u64, u64, u64, u64, vp, i32]
        _synth.synth_ivf_count.argtypes = [vp, vp, u64, u64, vp, i32]
        _synth.synth_ivf_count.restype = vp
        _synth.synth_ivf_fill.argtypes = [vp, vp, vp, vp, vp]
        _synth.synth_quantizer.argtypes = [u32, vp, vp]
        _synth.synth_quantizer.restype = C.c_int
        _synth.synth_queries.argtypes = [vp, u32, vp, vp, u32, vp, vp, vp, u64, u64, u32, dbl, u64, vp]
    return _synth


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class HostIndex:
    dim: int
    nbits: int
    centroids: np.ndarray      # K x dim float32
    codes: np.ndarray          # T uint32
    residuals: np.ndarray      # T x (nbits*dim/8) uint8 (flattened)
    doclens: np.ndarray        # N uint32
    ivf_offsets: np.ndarray    # K+1 uint64
    ivf_postings: np.ndarray   # P uint32
    bucket_cutoffs: np.ndarray  # 2^b-1 float32
    bucket_weights: np.ndarray  # 2^b float32
    passage_offsets: np.ndarray = field(default=None)  # N+1 uint64 (derived, index.cpp:7-10)

    def __post_init__(self):
        self.centroids = np.ascontiguousarray(self.centroids, dtype=np.float32)
        self.codes = np.ascontiguousarray(self.codes, dtype=np.uint32)
        self.residuals = np.ascontiguousarray(self.residuals, dtype=np.uint8).reshape(-1)
        self.doclens = np.ascontiguousarray(self.doclens, dtype=np.uint32)
        self.ivf_offsets = np.ascontiguousarray(self.ivf_offsets, dtype=np.uint64)
        self.ivf_postings = np.ascontiguousarray(self.ivf_postings, dtype=np.uint32)
        self.bucket_cutoffs = np.ascontiguousarray(self.bucket_cutoffs, dtype=np.float32)
        self.bucket_weights = np.ascontiguousarray(self.bucket_weights, dtype=np.float32)
        if self.passage_offsets is None:
            off = np.zeros(len(self.doclens) + 1, dtype=np.uint64)
            np.cumsum(self.doclens, dtype=np.uint64, out=off[1:])
            self.passage_offsets = off

    @property
    def num_centroids(self) -> int:
        return int(self.centroids.shape[0])

    @property
    def num_passages(self) -> int:
        return int(self.doclens.shape[0])

    @property
    def num_embeddings(self) -> int:
        return int(self.codes.shape[0])

    @property
    def bytes_per_token(self) -> int:
        return self.nbits * self.dim // 8

    def passage_codes(self, p: int) -> np.ndarray:
        o = self.passage_offsets
        return self.codes[int(o[p]):int(o[p + 1])]

    def nbytes(self) -> int:
        return sum(a.nbytes for a in (self.centroids, self.codes, self.residuals, self.doclens,
                                      self.ivf_offsets, self.ivf_postings))

    def save_npz(self, path) -> None:
        np.savez_compressed(path, dim=self.dim, nbits=self.nbits, centroids=self.centroids,
                            codes=self.codes, residuals=self.residuals, doclens=self.doclens,
                            ivf_offsets=self.ivf_offsets, ivf_postings=self.ivf_postings,
                            bucket_cutoffs=self.bucket_cutoffs, bucket_weights=self.bucket_weights)

    @classmethod
    def load_npz(cls, path) -> "HostIndex":
        z = np.load(path)
        return cls(int(z["dim"]), int(z["nbits"]), z["centroids"], z["codes"], z["residuals"],
                   z["doclens"], z["ivf_offsets"], z["ivf_postings"], z["bucket_cutoffs"],
                   z["bucket_weights"])


def build_inverted_list(codes: np.ndarray, doclens: np.ndarray, num_centroids: int,
                        threads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """build_inverted_list semantics (indexer.cpp:149-195), multithreaded C++."""
    lib = _lib()
    codes = np.ascontiguousarray(codes, dtype=np.uint32)
    doclens = np.ascontiguousarray(doclens, dtype=np.uint32)
    off = np.zeros(len(doclens) + 1, dtype=np.uint64)
    np.cumsum(doclens, dtype=np.uint64, out=off[1:])
    ivf_off = np.zeros(num_centroids + 1, dtype=np.uint64)
    st = lib.synth_ivf_count(_p(codes), _p(off), len(doclens), num_centroids, _p(ivf_off), threads)
    post = np.empty(int(ivf_off[-1]), dtype=np.uint32)
    lib.synth_ivf_fill(st, _p(codes), _p(off), _p(ivf_off), _p(post))
    return ivf_off, post


def quantizer(nbits: int) -> tuple[np.ndarray, np.ndarray]:
    cut = np.zeros((1 << nbits) - 1, dtype=np.float32)
    w = np.zeros(1 << nbits, dtype=np.float32)
    if _lib().synth_quantizer(nbits, _p(cut), _p(w)) != 0:
        raise ValueError(f"nbits {nbits} not in {{1,2,4}}")
    return cut, w


def generate_index(num_passages: int, num_centroids: int, dim: int = 128, nbits: int = 2,
                   mean_len: int = 64, spread: int = 16, repeat: float = 0.28, seed: int = 0,
                   threads: int = 0, pid_base: int = 0) -> HostIndex:
    """Synthetic index per SURVEY.md §8d: doclens uniform in [mean-spread,
    mean+spread], codes with a `repeat` chance of re-using an earlier code of
    the same passage (~0.72 postings/token), uniform residual bytes, and the
    fixed quantizer.  Fully determined by the arguments.  With pid_base > 0 the
    result is the passage range [pid_base, pid_base + num_passages) of the
    larger index with the same parameters (every stream is keyed by global
    passage id); its IVF is local to the range, with local ids."""
    lib = _lib()
    N, K = int(num_passages), int(num_centroids)
    cents = np.empty((K, dim), dtype=np.float32)
    lib.synth_centroids(K, dim, 11 + seed, _p(cents), threads)
    lo, hi = max(1, mean_len - spread), mean_len + spread
    doclens = np.empty(N, dtype=np.uint32)
    lib.synth_doclens(N, pid_base, lo, hi, 5 + seed, _p(doclens), threads)
    off = np.empty(N + 1, dtype=np.uint64)
    T = lib.synth_offsets(_p(doclens), N, _p(off))
    codes = np.empty(T, dtype=np.uint32)
    lib.synth_codes(_p(doclens), _p(off), N, pid_base, K, float(repeat), 99 + seed, _p(codes), threads)
    bpt = nbits * dim // 8
    res = np.empty(T * bpt, dtype=np.uint8)
    lib.synth_residuals(_p(off), N, pid_base, bpt, 7 + seed, _p(res), threads)
    ivf_off = np.zeros(K + 1, dtype=np.uint64)
    st = lib.synth_ivf_count(_p(codes), _p(off), N, K, _p(ivf_off), threads)
    post = np.empty(int(ivf_off[-1]), dtype=np.uint32)
    lib.synth_ivf_fill(st, _p(codes), _p(off), _p(ivf_off), _p(post))
    cut, w = quantizer(nbits)
    return HostIndex(dim, nbits, cents, codes, res, doclens, ivf_off, post, cut, w, off)


def generate_queries(index: HostIndex, num_queries: int, qlen: int = 32, noise: float = 0.03,
                     seed: int = 1234) -> np.ndarray:
    """[nq, qlen, dim] unit-norm query matrices near reconstructed corpus tokens."""
    lib = _lib()
    out = np.empty((num_queries, qlen, index.dim), dtype=np.float32)
    lib.synth_queries(_p(index.centroids), index.dim, _p(index.codes), _p(index.residuals), index.nbits,
                      _p(index.bucket_weights), _p(index.doclens), _p(index.passage_offsets),
                      index.num_passages, num_queries, qlen, float(noise), seed, _p(out))
    return out


# ---- on-disk format (FORMAT.md): host-side reader with an independent numpy
# implementation of the checksum (the GPU loader is DeviceIndex.open) -------------
_FNV_BASIS = np.uint64(0xCBF29CE484222325)
_FNV_PRIME = np.uint64(0x100000001B3)
_FILES = ("centroids.f32", "codes.u32", "residuals.bin", "doclens.u32", "ivf_offsets.u64", "ivf_postings.u32")


def fnv_digest(buf: bytes | np.ndarray) -> int:
    """FORMAT.md digest: 64 KiB blocks, word i of a block -> lane i % 32,
    FNV-1a 64 over 64-bit little-endian words (tail zero-padded), lanes folded
    into the block digest, block digests + byte length into the file digest."""
    raw = np.frombuffer(bytes(buf) if not isinstance(buf, np.ndarray) else np.ascontiguousarray(buf).tobytes(),
                        dtype=np.uint8)
    nbytes = raw.size
    block = 64 * 1024
    nb = (nbytes + block - 1) // block
    with np.errstate(over="ignore"):
        digests = []
        if nb:
            padded = np.zeros(nb * block, dtype=np.uint8)
            padded[:nbytes] = raw
            words = padded.view("<u8").reshape(nb, block // 8 // 32, 32)  # [block, step, lane]
            nwords = np.full(nb, block // 8, dtype=np.int64)
            nwords[-1] = (nbytes - (nb - 1) * block + 7) // 8
            lanes = np.full((nb, 32), _FNV_BASIS, dtype=np.uint64)
            for s in range(words.shape[1]):
                active = (s * 32 + np.arange(32))[None, :] < nwords[:, None]
                lanes = np.where(active, (lanes ^ words[:, s, :]) * _FNV_PRIME, lanes)
            d = np.full(nb, _FNV_BASIS, dtype=np.uint64)
            for l in range(32):
                d = (d ^ lanes[:, l]) * _FNV_PRIME
            digests = list(d)
        h = _FNV_BASIS
        for x in digests:
            h = (h ^ np.uint64(x)) * _FNV_PRIME
        h = (h ^ np.uint64(nbytes)) * _FNV_PRIME
    return int(h)


def load_index_host(path, verify: bool = True) -> HostIndex:
    """Read an index written by save_index (FORMAT.md) into host memory."""
    import json
    import os

    from .api import ErrorCode, PlaidError

    with open(os.path.join(path, "manifest.json")) as f:
        m = json.load(f)
    if m.get("format_version") != 1:
        raise PlaidError(ErrorCode.UnsupportedVersion, f"format_version {m.get('format_version')}")
    arrays = {}
    for name, dt in zip(_FILES, ("<f4", "<u4", "u1", "<u4", "<u8", "<u4")):
        data = np.fromfile(os.path.join(path, name), dtype=np.uint8)
        if verify and f"{fnv_digest(data):016x}" != m["checksums"][name]:
            raise PlaidError(ErrorCode.ChecksumMismatch, f"{name}: checksum mismatch")
        arrays[name] = data.view(dt)
    dim, K = int(m["dim"]), int(m["num_centroids"])
    cut = np.array(m["bucket_cutoffs_bits"], dtype=np.uint32).view(np.float32)
    wts = np.array(m["bucket_weights_bits"], dtype=np.uint32).view(np.float32)
    return HostIndex(dim, int(m["nbits"]), arrays["centroids.f32"].reshape(K, dim), arrays["codes.u32"],
                     arrays["residuals.bin"], arrays["doclens.u32"], arrays["ivf_offsets.u64"],
                     arrays["ivf_postings.u32"], cut, wts)

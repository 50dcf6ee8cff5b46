"""CPU oracles for the PLAID search path — TEST INFRASTRUCTURE ONLY.

Two implementations behind one Python interface:
  * "port": oracle/liboracle.so, the plain-C restatement (plaid_oracle.c),
    single-threaded, every function citing the reference file:line it follows;
  * "ref":  oracle/_ref/liblir_ref.so, the UNMODIFIED reference sources
    (/root/reference/proj/src) compiled by oracle/Makefile with a thin extern "C"
    shim (ref_shim.cpp).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/--impl
reference legs may use this package, and only as the checker or the timed CPU
baseline.  The product (paper_2205_09707_b200) never imports it.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "liblir_ref.so"
# the same reference sources at -O3 -march=native of the build host (Sapphire
# Rapids here): the timed CPU baseline when the running host has every ISA
# extension that build may use (native_isa_ok), else the portable build
REF_NATIVE_SO = HERE / "_ref" / "liblir_ref_native.so"
REF_NATIVE_ISA = HERE / "_ref" / "native_isa.txt"

u8p, u32p, u64p, f32p = (C.POINTER(C.c_uint8), C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                         C.POINTER(C.c_float))


class OrcIndex(C.Structure):
    _fields_ = [("dim", C.c_uint32), ("nbits", C.c_uint32), ("num_centroids", C.c_uint64),
                ("num_passages", C.c_uint64), ("num_embeddings", C.c_uint64),
                ("centroids", f32p), ("codes", u32p), ("residuals", u8p), ("doclens", u32p),
                ("passage_offsets", u64p), ("ivf_offsets", u64p), ("ivf_postings", u32p),
                ("bucket_cutoffs", f32p), ("bucket_weights", f32p)]


class OrcParams(C.Structure):
    _fields_ = [("k", C.c_uint64), ("nprobe", C.c_uint64), ("t_cs", C.c_float), ("ndocs", C.c_uint64),
                ("disable_filter", C.c_int32)]


class OrcTrace(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "stage1_candidates", "stage2_out", "stage3_out", "final_out", "centroid_matmul_count",
        "stage2_rows_gathered", "stage3_rows_gathered", "decompressed_passages")]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status          # lir::ErrorCode + 1
        self.code = status - 1        # lir::ErrorCode value


def _p(a, t):
    return None if a is None else a.ctypes.data_as(C.POINTER(t))


def _orc_index(h) -> OrcIndex:
    return OrcIndex(h.dim, h.nbits, h.num_centroids, h.num_passages, h.num_embeddings,
                    _p(h.centroids, C.c_float), _p(h.codes, C.c_uint32), _p(h.residuals, C.c_uint8),
                    _p(h.doclens, C.c_uint32), _p(h.passage_offsets, C.c_uint64),
                    _p(h.ivf_offsets, C.c_uint64), _p(h.ivf_postings, C.c_uint32),
                    _p(h.bucket_cutoffs, C.c_float), _p(h.bucket_weights, C.c_float))


def _params(p, disable_filter=False) -> OrcParams:
    return OrcParams(int(p.k), int(p.nprobe), float(p.t_cs), int(p.ndocs), int(bool(disable_filter)))


class CpuOracle:
    """Same method surface as paper_2205_09707_b200.Searcher, on HostIndex."""

    def __init__(self, kind: str):
        self.kind = kind
        path = {"port": PORT_SO, "ref": REF_SO, "ref_native": REF_NATIVE_SO}[kind]
        if not path.exists():
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.path = path
        self.lib = C.CDLL(str(path))
        self.pre = "orc_" if kind == "port" else "ref_"
        self._ref_handles = {}
        L = self.lib
        vp = C.c_void_p
        u64 = C.c_uint64
        self._fn("last_error", C.c_char_p, [])
        if kind == "port":
            self._fn("search", C.c_int, [C.POINTER(OrcIndex), f32p, u64, u64, C.POINTER(OrcParams), u32p, f32p,
                                         u64p, C.POINTER(OrcTrace)])
            self._fn("centroid_interaction", C.c_int, [C.POINTER(OrcIndex), f32p, u64, u32p, u64, u8p, f32p, u64p])
            self._fn("rank_final", C.c_int, [C.POINTER(OrcIndex), f32p, u64, u32p, u64, u64, u32p, f32p, u64p])
            self._fn("reconstruct", C.c_int, [u32p, u64, u8p, f32p, C.c_uint32, C.c_uint32, f32p, f32p])
        else:
            self._fn("index_build", vp, [C.POINTER(OrcIndex), C.POINTER(C.c_int)])
            self._fn("index_free", None, [vp])
            self._fn("index_validate", C.c_int, [vp])
            self._fn("search", C.c_int, [vp, f32p, u64, u64, C.POINTER(OrcParams), C.c_int, u32p, f32p, u64p,
                                         C.POINTER(OrcTrace), C.POINTER(C.c_double)])
            self._fn("search_many", C.c_int, [vp, f32p, u64, u64, u64, C.POINTER(OrcParams), C.c_int, C.c_int,
                                              u32p, f32p, u64p, C.POINTER(C.c_double)])
            self._fn("centroid_interaction", C.c_int, [vp, f32p, u64, u32p, u64, u8p, f32p, u64p])
            self._fn("rank_final", C.c_int, [vp, f32p, u64, u32p, u64, u64, u32p, f32p, u64p])
            self._fn("reconstruct", C.c_int, [u32p, u64, u8p, f32p, u64, C.c_uint32, C.c_uint32, f32p, f32p, f32p])
            self._fn("build_inverted_list", C.c_int, [u32p, u64, u32p, u64, u64, u64p, u32p, u64, u64p])
            self._fn("build_index", vp, [f32p, u32p, u64, u64, C.c_uint32, u64, u64, u64, C.c_int,
                                         C.POINTER(C.c_int)])
            self._fn("index_sizes", None, [vp, u64p])
            self._fn("index_export", None, [vp, f32p, u32p, u8p, u32p, u64p, u32p, f32p, f32p])
        self._fn("validate_query", C.c_int, [f32p, u64, u64, u64])
        self._fn("validate_params", C.c_int, [C.POINTER(OrcParams), u64])
        self._fn("default_params_for_k", None, [u64, C.POINTER(OrcParams)])
        self._fn("stage3_width", u64, [C.POINTER(OrcParams)])
        self._fn("lut_build", C.c_int, [C.c_uint32, u8p])
        self._fn("pack_residual", C.c_int, [u8p, u64, C.c_uint32, u8p])
        self._fn("unpack_via_lut", C.c_int, [u8p, u64, C.c_uint32, u8p])
        self._fn("compute_centroid_scores", C.c_int, [f32p, u64, u64, f32p, u64, f32p, f32p])
        self._fn("generate_candidates", C.c_int, [f32p, u64, u64, u64p, u32p, u64, u64, u32p, u64p])
        self._fn("prune_centroids", None, [f32p, u64, C.c_float, u8p])
        self._fn("select_top", C.c_int, [u32p, f32p, u64, u64, u32p, f32p, u64p])
        self._fn("maxsim_packed", C.c_int, [f32p, u64, u64p, u64, f32p])
        self._fn("maxsim_embeddings", C.c_int, [f32p, u64, u64, f32p, u64p, u64, f32p])
        del L

    def _fn(self, name, res, args):
        f = getattr(self.lib, self.pre + name)
        f.restype = res
        f.argtypes = args
        setattr(self, "_" + name, f)

    def _check(self, st: int) -> None:
        if st:
            raise OracleError(st, self._last_error().decode(errors="replace"))

    # ------------------------------------------------------------ index handles (ref)
    def ref_handle(self, index):
        key = id(index)
        ent = self._ref_handles.get(key)
        if ent is None or ent[1] is not index:
            st = C.c_int()
            d = _orc_index(index)
            h = self._index_build(C.byref(d), C.byref(st))
            self._check(st.value)
            ent = (h, index)
            self._ref_handles[key] = ent
        return ent[0]

    def release(self, index) -> None:
        ent = self._ref_handles.pop(id(index), None)
        if ent is not None:
            self._index_free(ent[0])

    def _ix(self, index):
        if self.kind == "port":
            d = _orc_index(index)
            self._keep = d
            return C.byref(d)
        return self.ref_handle(index)

    # ------------------------------------------------------------ pipeline
    def search(self, index, q, params, disable_filter=False, threads=1, times=None):
        q = np.ascontiguousarray(q, dtype=np.float32)
        k = max(int(params.k), 1)
        ids = np.zeros(k, dtype=np.uint32)
        sc = np.zeros(k, dtype=np.float32)
        n = C.c_uint64()
        tr = OrcTrace()
        p = _params(params, disable_filter)
        rows, dim = (q.shape if q.ndim == 2 else (0, 0))
        if self.kind == "port":
            st = self._search(self._ix(index), _p(q, C.c_float), rows, dim, C.byref(p), _p(ids, C.c_uint32),
                              _p(sc, C.c_float), C.byref(n), C.byref(tr))
        else:
            tm = (C.c_double * 7)()
            st = self._search(self._ix(index), _p(q, C.c_float), rows, dim, C.byref(p), int(threads),
                              _p(ids, C.c_uint32), _p(sc, C.c_float), C.byref(n), C.byref(tr), tm)
            if times is not None:
                times[:] = list(tm)
        self._check(st)
        trace = {f: getattr(tr, f) for f, _ in OrcTrace._fields_}
        return ids[: n.value].copy(), sc[: n.value].copy(), trace

    def search_many(self, index, qs, params, mode: int, threads: int):
        """ref only: mode 0 latency (threads per query), 1 throughput (threads x 1)."""
        qs = np.ascontiguousarray(qs, dtype=np.float32)
        nq, rows, dim = qs.shape
        k = int(params.k)
        ids = np.zeros((nq, k), dtype=np.uint32)
        sc = np.zeros((nq, k), dtype=np.float32)
        n = np.zeros(nq, dtype=np.uint64)
        lat = np.zeros(nq, dtype=np.float64)
        p = _params(params)
        self._check(self._search_many(self.ref_handle(index), _p(qs, C.c_float), nq, rows, dim, C.byref(p),
                                      mode, threads, _p(ids, C.c_uint32), _p(sc, C.c_float),
                                      _p(n, C.c_uint64), _p(lat, C.c_double)))
        return ids, sc, n, lat

    def validate_index(self, index) -> None:
        self._check(self._index_validate(self.ref_handle(index)))

    def compute_centroid_scores(self, index, q):
        q = np.ascontiguousarray(q, dtype=np.float32)
        K = index.num_centroids
        S = np.zeros((K, q.shape[0]), dtype=np.float32)
        mx = np.zeros(K, dtype=np.float32)
        self._check(self._compute_centroid_scores(_p(q, C.c_float), q.shape[0], q.shape[1],
                                                  _p(index.centroids, C.c_float), K, _p(S, C.c_float),
                                                  _p(mx, C.c_float)))
        return S, mx

    def generate_candidates(self, index, S, nprobe):
        S = np.ascontiguousarray(S, dtype=np.float32)
        out = np.zeros(max(index.num_passages, 1), dtype=np.uint32)
        n = C.c_uint64()
        self._check(self._generate_candidates(_p(S, C.c_float), S.shape[0], S.shape[1],
                                              _p(index.ivf_offsets, C.c_uint64), _p(index.ivf_postings, C.c_uint32),
                                              int(nprobe), index.num_passages, _p(out, C.c_uint32), C.byref(n)))
        return out[: n.value].copy()

    def prune_centroids(self, row_max, t_cs):
        mx = np.ascontiguousarray(row_max, dtype=np.float32)
        keep = np.zeros(mx.size, dtype=np.uint8)
        self._prune_centroids(_p(mx, C.c_float), mx.size, float(t_cs), _p(keep, C.c_uint8))
        return keep

    def centroid_interaction(self, index, cand, S, mask):
        cand = np.ascontiguousarray(cand, dtype=np.uint32)
        S = np.ascontiguousarray(S, dtype=np.float32)
        m = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)
        out = np.zeros(max(cand.size, 1), dtype=np.float32)
        rows = C.c_uint64()
        self._check(self._centroid_interaction(self._ix(index), _p(S, C.c_float), S.shape[1], _p(cand, C.c_uint32),
                                               cand.size, _p(m, C.c_uint8), _p(out, C.c_float), C.byref(rows)))
        return out[: cand.size].copy(), int(rows.value)

    def select_top(self, ids, scores, n):
        ids = np.ascontiguousarray(ids, dtype=np.uint32)
        sc = np.ascontiguousarray(scores, dtype=np.float32)
        m = max(min(int(n), ids.size), 1)
        oi = np.zeros(m, dtype=np.uint32)
        os_ = np.zeros(m, dtype=np.float32)
        cnt = C.c_uint64()
        self._check(self._select_top(_p(ids, C.c_uint32), _p(sc, C.c_float), ids.size, int(n),
                                     _p(oi, C.c_uint32), _p(os_, C.c_float), C.byref(cnt)))
        return oi[: cnt.value].copy(), os_[: cnt.value].copy()

    def rank_final(self, index, cand, q, k):
        cand = np.ascontiguousarray(cand, dtype=np.uint32)
        q = np.ascontiguousarray(q, dtype=np.float32)
        m = max(min(int(k), cand.size), 1)
        oi = np.zeros(m, dtype=np.uint32)
        os_ = np.zeros(m, dtype=np.float32)
        cnt = C.c_uint64()
        self._check(self._rank_final(self._ix(index), _p(q, C.c_float), q.shape[0], _p(cand, C.c_uint32),
                                     cand.size, int(k), _p(oi, C.c_uint32), _p(os_, C.c_float), C.byref(cnt)))
        return oi[: cnt.value].copy(), os_[: cnt.value].copy()

    def reconstruct(self, index, codes, residuals):
        codes = np.ascontiguousarray(codes, dtype=np.uint32)
        res = np.ascontiguousarray(residuals, dtype=np.uint8).reshape(-1)
        out = np.zeros((codes.size, index.dim), dtype=np.float32)
        if self.kind == "port":
            st = self._reconstruct(_p(codes, C.c_uint32), codes.size, _p(res, C.c_uint8),
                                   _p(index.centroids, C.c_float), index.dim, index.nbits,
                                   _p(index.bucket_weights, C.c_float), _p(out, C.c_float))
        else:
            st = self._reconstruct(_p(codes, C.c_uint32), codes.size, _p(res, C.c_uint8),
                                   _p(index.centroids, C.c_float), index.num_centroids, index.dim, index.nbits,
                                   _p(index.bucket_cutoffs, C.c_float), _p(index.bucket_weights, C.c_float),
                                   _p(out, C.c_float))
        self._check(st)
        return out

    def lut_build(self, nbits):
        t = np.zeros(256 * 8, dtype=np.uint8)
        self._check(self._lut_build(nbits, _p(t, C.c_uint8)))
        return t[: 256 * (8 // nbits)].reshape(256, 8 // nbits)

    def pack_residual(self, idx, nbits):
        idx = np.ascontiguousarray(idx, dtype=np.uint8)
        out = np.zeros(max(1, idx.size), dtype=np.uint8)
        self._check(self._pack_residual(_p(idx, C.c_uint8), idx.size, nbits, _p(out, C.c_uint8)))
        return out[: idx.size * nbits // 8]

    def unpack_via_lut(self, packed, nbits):
        pk = np.ascontiguousarray(packed, dtype=np.uint8).reshape(-1)
        out = np.zeros(max(1, pk.size * 8), dtype=np.uint8)
        self._check(self._unpack_via_lut(_p(pk, C.c_uint8), pk.size, nbits, _p(out, C.c_uint8)))
        return out[: pk.size * (8 // nbits)]

    def maxsim_packed(self, scores, offsets):
        S = np.ascontiguousarray(scores, dtype=np.float32)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        np_ = off.size - 1
        out = np.zeros(max(np_, 1), dtype=np.float32)
        self._check(self._maxsim_packed(_p(S, C.c_float), S.shape[1], _p(off, C.c_uint64), np_, _p(out, C.c_float)))
        return out[:np_]

    def maxsim_embeddings(self, q, emb, offsets):
        q = np.ascontiguousarray(q, dtype=np.float32)
        e = np.ascontiguousarray(emb, dtype=np.float32)
        off = np.ascontiguousarray(offsets, dtype=np.uint64)
        np_ = off.size - 1
        out = np.zeros(max(np_, 1), dtype=np.float32)
        self._check(self._maxsim_embeddings(_p(q, C.c_float), q.shape[0], q.shape[1], _p(e, C.c_float),
                                            _p(off, C.c_uint64), np_, _p(out, C.c_float)))
        return out[:np_]

    def validate_query(self, q, index_dim):
        q = np.ascontiguousarray(q, dtype=np.float32)
        rows, dim = (q.shape if q.ndim == 2 else (0, 0))
        self._check(self._validate_query(_p(q, C.c_float), rows, dim, int(index_dim)))

    def validate_params(self, params, K):
        p = _params(params)
        self._check(self._validate_params(C.byref(p), int(K)))

    def default_params_for_k(self, k):
        p = OrcParams()
        self._default_params_for_k(int(k), C.byref(p))
        return (int(p.k), int(p.nprobe), float(p.t_cs), int(p.ndocs))

    def stage3_width(self, params):
        p = _params(params)
        return int(self._stage3_width(C.byref(p)))

    # ------------------------------------------------------------ ref-only helpers
    def build_inverted_list(self, codes, doclens, K):
        codes = np.ascontiguousarray(codes, dtype=np.uint32)
        doclens = np.ascontiguousarray(doclens, dtype=np.uint32)
        off = np.zeros(K + 1, dtype=np.uint64)
        cap = codes.size
        post = np.zeros(max(cap, 1), dtype=np.uint32)
        P = C.c_uint64()
        self._check(self._build_inverted_list(_p(codes, C.c_uint32), codes.size, _p(doclens, C.c_uint32),
                                              doclens.size, K, _p(off, C.c_uint64), _p(post, C.c_uint32), cap,
                                              C.byref(P)))
        return off, post[: P.value].copy()

    def build_index(self, data, doclens, dim, nbits, K, iters=5, seed=42, threads=0):
        """The reference's own offline build (k-means), exported as arrays."""
        data = np.ascontiguousarray(data, dtype=np.float32)
        doclens = np.ascontiguousarray(doclens, dtype=np.uint32)
        st = C.c_int()
        h = self._build_index(_p(data, C.c_float), _p(doclens, C.c_uint32), doclens.size, dim, nbits, K, iters,
                              seed, threads, C.byref(st))
        self._check(st.value)
        sz = np.zeros(6, dtype=np.uint64)
        self._index_sizes(h, _p(sz, C.c_uint64))
        d, b, K_, N_, T_, P_ = (int(x) for x in sz)
        cents = np.zeros((K_, d), dtype=np.float32)
        codes = np.zeros(T_, dtype=np.uint32)
        res = np.zeros(T_ * b * d // 8, dtype=np.uint8)
        dl = np.zeros(N_, dtype=np.uint32)
        ivo = np.zeros(K_ + 1, dtype=np.uint64)
        post = np.zeros(max(P_, 1), dtype=np.uint32)
        cut = np.zeros((1 << b) - 1, dtype=np.float32)
        w = np.zeros(1 << b, dtype=np.float32)
        self._index_export(h, _p(cents, C.c_float), _p(codes, C.c_uint32), _p(res, C.c_uint8), _p(dl, C.c_uint32),
                           _p(ivo, C.c_uint64), _p(post, C.c_uint32), _p(cut, C.c_float), _p(w, C.c_float))
        self._index_free(h)
        return dict(dim=d, nbits=b, centroids=cents, codes=codes, residuals=res, doclens=dl,
                    ivf_offsets=ivo, ivf_postings=post[:P_], bucket_cutoffs=cut, bucket_weights=w)


_cache = {}


def get(kind: str) -> CpuOracle:
    if kind not in _cache:
        _cache[kind] = CpuOracle(kind)
    return _cache[kind]


def available(kind: str) -> bool:
    if kind == "ref_native":
        return REF_NATIVE_SO.exists() and native_isa_ok()
    return (PORT_SO if kind == "port" else REF_SO).exists()


def _cpu_flags() -> set:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("flags"):
                return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def native_isa_ok() -> bool:
    """True when this host has every SIMD extension of the host that built
    liblir_ref_native.so (recorded next to it by oracle/Makefile)."""
    if not REF_NATIVE_ISA.exists():
        return False
    need = set(REF_NATIVE_ISA.read_text().split())
    return need <= _cpu_flags()


def timed_reference() -> tuple:
    """(oracle, flags note) for the timed CPU baseline: the -march=native build
    when this host can run it, else the portable -march=x86-64-v3 build."""
    if available("ref_native"):
        return get("ref_native"), "g++ -O3 -march=native (build host: " + \
            (HERE / "_ref" / "native_march.txt").read_text().strip() + ") -ffp-contract=off"
    return get("ref"), "g++ -O3 -march=x86-64-v3 -ffp-contract=off (host lacks the native build's ISA)"

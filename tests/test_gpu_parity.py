"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on
identical index bytes and queries.  Integer outputs and, in EXACT score mode,
every fp32 score must be bit-identical to the reference arithmetic."""
import os

import numpy as np
import pytest

import paper_2205_09707_b200 as P

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def small():
    h = P.generate_index(4000, 512, dim=128, nbits=2, mean_len=40, seed=1)
    qs = P.generate_queries(h, 6, seed=11)
    idx = P.DeviceIndex.from_host(h)
    return h, qs, idx, P.Searcher(idx)


@pytest.mark.parametrize("k", [1, 10, 100, 1000])
def test_search_bit_exact(small, port, k):
    h, qs, idx, s = small
    p = P.default_params_for_k(k)
    for q in qs:
        got = s.search(q, p)
        ids, sc, tr = port.search(h, q, p)
        assert np.array_equal(got.topk.passage_ids, ids)
        assert np.array_equal(bits(got.topk.scores), bits(sc))
        assert got.trace.counters() == tr


def test_stages_bit_exact(small, port):
    h, qs, idx, s = small
    q = qs[0]
    S, mx = s.compute_centroid_scores(q)
    S0, mx0 = port.compute_centroid_scores(h, q)
    assert np.array_equal(bits(S), bits(S0))
    assert np.array_equal(mx, mx0)
    for nprobe in (1, 2, 4, 7, 32, 33, h.num_centroids):
        assert np.array_equal(s.generate_candidates(S0, nprobe), port.generate_candidates(h, S0, nprobe)), nprobe
    c1 = port.generate_candidates(h, S0, 4)
    for t_cs in (-1.0, 0.2, 0.4, 0.5, 1.0):
        keep = port.prune_centroids(mx0, t_cs)
        assert np.array_equal(s.prune_centroids(mx0, t_cs), keep)
        g, gr = s.centroid_interaction(c1, S0, keep)
        o, orr = port.centroid_interaction(h, c1, S0, keep)
        assert np.array_equal(bits(g), bits(o)) and gr == orr, t_cs
    g, gr = s.centroid_interaction(c1, S0, None)
    o, orr = port.centroid_interaction(h, c1, S0, None)
    assert np.array_equal(bits(g), bits(o)) and gr == orr
    for n in (1, 10, 256, 4096, len(c1), len(c1) + 5):
        a = s.select_top(c1, o, n)
        b = port.select_top(c1, o, n)
        assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1])), n
    a = s.rank_final(c1[:300], q, 100)
    b = port.rank_final(h, c1[:300], q, 100)
    assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1]))


def test_codec_bit_exact(small, port):
    h, qs, idx, s = small
    t = np.arange(0, 3000, 7)
    res = h.residuals.reshape(h.num_embeddings, -1)[t]
    assert np.array_equal(bits(s.reconstruct(h.codes[t], res)), bits(port.reconstruct(h, h.codes[t], res)))
    pk = np.arange(256, dtype=np.uint8)
    for b in (1, 2, 4):
        assert np.array_equal(s.unpack_via_lut(pk, b), port.unpack_via_lut(pk, b))


def test_disable_filter(small, port):
    h, qs, idx, s = small
    p = P.default_params_for_k(100)
    got = s.search(qs[1], p, P.SearchOptions(disable_filter=True))
    ids, sc, tr = port.search(h, qs[1], p, disable_filter=True)
    assert np.array_equal(got.topk.passage_ids, ids)
    assert np.array_equal(bits(got.topk.scores), bits(sc))
    assert got.trace.counters() == tr


@pytest.mark.parametrize("n,keep", [(20000, 4096), (100000, 1000), (100000, 9000), (50000, 60000), (9000, 8200)])
def test_select_top_large_ties(port, n, keep):
    """Radix-select + global sort paths, with heavy score ties (tie -> lower pid)."""
    rng = np.random.default_rng(n + keep)
    s = P.Searcher(None)
    ids = rng.permutation(n * 3)[:n].astype(np.uint32)
    sc = rng.choice(np.array([0.0, -0.0, 1.5, 2.25, -3.0, 7.0], dtype=np.float32), size=n)
    sc[: n // 3] = rng.standard_normal(n // 3).astype(np.float32)
    a = s.select_top(ids, sc, keep)
    b = port.select_top(ids, sc, keep)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1])


def compose_with_scores(port, h, q, S, mx, p):
    """The reference pipeline (pipeline.cpp:232-283) run by the oracle stage by
    stage, but on a given centroid-score table S (e.g. the tensor-core one)."""
    c1 = port.generate_candidates(h, S, p.nprobe)
    keep = port.prune_centroids(mx, p.t_cs)
    s2, r2 = port.centroid_interaction(h, c1, S, keep)
    k2, _ = port.select_top(c1, s2, p.ndocs)
    s3, r3 = port.centroid_interaction(h, k2, S, None)
    k3, _ = port.select_top(k2, s3, P.stage3_width(p))
    ids, sc = port.rank_final(h, k3, q, p.k)
    return ids, sc, dict(stage1_candidates=len(c1), stage2_out=len(k2), stage3_out=len(k3), final_out=len(ids),
                         centroid_matmul_count=1, stage2_rows_gathered=r2, stage3_rows_gathered=r3,
                         decompressed_passages=len(k3))


@pytest.fixture(scope="module")
def tensor_searcher(small):
    h, qs, idx, _ = small
    return P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)


def test_tensor_scores_accuracy(small, tensor_searcher, port):
    """tcgen05 3xTF32 S_cq vs the in-order fp32 reference dot products."""
    h, qs, idx, _ = small
    for q in qs:
        S, mx = tensor_searcher.compute_centroid_scores(q)
        S0, mx0 = port.compute_centroid_scores(h, q)
        assert np.abs(S - S0).max() < 5e-6
        assert np.abs(mx - mx0).max() < 5e-6


@pytest.mark.parametrize("k", [10, 100, 1000])
def test_tensor_search_consistent(small, tensor_searcher, port, k):
    """Given the tensor-core S, stages 1-3 are bit-exact with the oracle run on
    that S (every trace counter equal) and the tensor-core stage 4 (S-row
    reuse + split-bf16 residual products) stays within the north_star
    tolerance: MaxSim within 1e-4 relative, top-k equal except near-ties."""
    from oracle.compare import check_tensor_search

    h, qs, idx, _ = small
    p = P.default_params_for_k(k)
    for q in qs:
        S, mx = tensor_searcher.compute_centroid_scores(q)
        got = tensor_searcher.search(q, p)
        rep = check_tensor_search(port, h, q, p, got.topk.passage_ids, got.topk.scores, S,
                                  got_counters=got.trace.counters())
        assert rep.ok, rep.as_dict()
        assert rep.max_rel_score_err < 2e-5  # measured ~1e-6; the bar is 1e-4


def test_tensor_stage4_scores(small, tensor_searcher, port):
    """The tensor stage-4 MaxSim of every finalist vs the exact reference
    MaxSim (disable_filter sends all stage-1 candidates through stage 4)."""
    h, qs, idx, _ = small
    p = P.SearchParams(400, 2, 0.5, 400)
    for q in qs[:3]:
        got = tensor_searcher.search(q, p, P.SearchOptions(disable_filter=True))
        ids, ex = port.rank_final(h, got.topk.passage_ids, q, len(got.topk.passage_ids))
        exact = dict(zip(ids.tolist(), ex.tolist()))
        err = max(abs(float(s) - exact[int(i)]) / abs(exact[int(i)])
                  for i, s in zip(got.topk.passage_ids, got.topk.scores))
        assert err < 2e-5, err


def test_merge_topk(port):
    rng = np.random.default_rng(5)
    s = P.Searcher(None)
    G, k = 4, 100
    pids = np.zeros((G, k), np.uint32)
    sc = np.zeros((G, k), np.float32)
    counts = np.array([100, 37, 0, 100], np.uint64)
    allp, alls = [], []
    for g in range(G):
        c = int(counts[g])
        p = (rng.permutation(10000)[:c] + g * 10000).astype(np.uint32)
        v = rng.standard_normal(c).astype(np.float32)
        pids[g, :c], sc[g, :c] = p, v
        allp.append(p), alls.append(v)
    a = s.merge_topk(pids, sc, counts, k)
    b = port.select_top(np.concatenate(allp), np.concatenate(alls), k)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_golden_gpu(golden):
    """CUDA path (EXACT mode, through the C ABI) against the reference's own
    golden outputs (tests/golden/make_golden.py)."""
    idx = P.DeviceIndex.from_host(golden.index, validate=True)
    s = P.Searcher(idx)
    for qi, q in enumerate(golden.queries):
        for pi, p in enumerate(golden.params):
            r = s.search(q, p)
            e_ids, e_bits, e_tr = golden.expected(qi, pi)
            assert np.array_equal(r.topk.passage_ids, e_ids), (golden.name, qi, pi)
            assert np.array_equal(bits(r.topk.scores), e_bits), (golden.name, qi, pi)
            assert r.trace.counters() == e_tr, (golden.name, qi, pi)


@pytest.mark.parametrize("params", [(10, 3, 0.3, 64), (50, 8, -1.0, 800), (7, 2, 0.9, 16), (20, 5, 0.45, 20),
                                    (100, 512, 0.2, 4000)])
def test_search_params_sweep_gpu(small, port, params):
    """Stage 2 through the kept-list path and its long-list fallback (t_cs=-1)."""
    h, qs, idx, s = small
    p = P.SearchParams(*params)
    for q in qs[:3]:
        got = s.search(q, p)
        ids, sc, tr = port.search(h, q, p)
        assert np.array_equal(got.topk.passage_ids, ids)
        assert np.array_equal(bits(got.topk.scores), bits(sc))
        assert got.trace.counters() == tr


def test_saturated_multiplicity(port):
    """A passage repeating one code > 255 times: the gathered-row counter
    still matches the reference (saturated ivf_mult entries are recounted)."""
    rng = np.random.default_rng(3)
    K, dim = 16, 128
    C = rng.standard_normal((K, dim)).astype(np.float32)
    C /= np.linalg.norm(C, axis=1, keepdims=True)
    doclens = np.array([300, 20, 40, 300], np.uint32)
    codes = np.concatenate([np.full(300, 3), rng.integers(0, K, 20), rng.integers(0, K, 40),
                            np.concatenate([np.full(280, 7), rng.integers(0, K, 20)])]).astype(np.uint32)
    ivo, post = P.build_inverted_list(codes, doclens, K)
    cut, w = P.hostindex.quantizer(2)
    res = rng.integers(0, 256, size=codes.size * 32, dtype=np.uint8)
    h = P.HostIndex(dim, 2, C, codes, res, doclens, ivo, post, cut, w)
    s = P.Searcher(P.DeviceIndex.from_host(h, validate=True))
    q = np.stack([C[3], C[7]] + [C[i % K] for i in range(30)]).astype(np.float32)
    for prm in (P.SearchParams(4, 2, 0.5, 4), P.SearchParams(4, 16, -1.0, 16), P.SearchParams(2, 4, 0.9, 4)):
        got = s.search(q, prm)
        ids, sc, tr = port.search(h, q, prm)
        assert np.array_equal(got.topk.passage_ids, ids)
        assert np.array_equal(bits(got.topk.scores), bits(sc))
        assert got.trace.counters() == tr


def test_lir_dropin_binary():
    """The drop-in demonstration: reference `lir` code (compiled reference
    sources) swaps lir::search for plaid_lir::Engine::search unchanged, and
    both return identical ids, score bits and trace counters."""
    import subprocess
    from pathlib import Path

    exe = Path(__file__).resolve().parents[1] / "oracle" / "_ref" / "lir_dropin"
    if not exe.exists():
        pytest.skip("oracle/_ref/lir_dropin not built (needs the reference sources at build time)")
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("OK")


def test_stage2_select_massive_ties(port):
    """Stage-2 select when the ndocs boundary falls among > 8192 equal (zero)
    scores: the histogram select's one-CTA radix fallback (select.cu)."""
    h = P.generate_index(40000, 1024, dim=128, nbits=2, mean_len=20, spread=8, seed=9)
    qs = P.generate_queries(h, 2, seed=5)
    s = P.Searcher(P.DeviceIndex.from_host(h))
    for prm in (P.SearchParams(50, 256, 0.9, 30000), P.SearchParams(50, 64, 0.95, 9000),
                P.SearchParams(10, 16, 0.3, 200)):
        for q in qs:
            got = s.search(q, prm)
            ids, sc, tr = port.search(h, q, prm)
            assert tr["stage1_candidates"] > 8192 or prm.ndocs == 200
            assert np.array_equal(got.topk.passage_ids, ids)
            assert np.array_equal(bits(got.topk.scores), bits(sc))
            assert got.trace.counters() == tr


@pytest.mark.parametrize("G", [2, 3, 8])
def test_global_exact_shards_bit_exact(port, G):
    """Global-exact passage sharding with G shards resident on
    one GPU: the three device phases + key exchanges + merge reproduce the
    UNSHARDED reference search bit for bit, and the summed trace counters
    equal its StageTrace."""
    import torch

    from paper_2205_09707_b200.sharded import search_local_shards, shard_range

    N, K = 6000, 512
    whole = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
    qs = P.generate_queries(whole, 4, seed=21)
    shards = []
    for g in range(G):
        a, b = shard_range(N, G, g)
        hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
        ix = P.DeviceIndex.from_host_at(hs, pid_base=a)
        shards.append((ix, P.Searcher(ix, score_mode=P.ScoreMode.EXACT)))
    ss = [s for _, s in shards]
    cases = [P.default_params_for_k(k) for k in (10, 100)] + [P.SearchParams(20, 8, -1.0, 300),
                                                               P.SearchParams(50, 4, 0.3, 64)]
    for p in cases:
        for q in qs:
            dq = torch.from_numpy(q.copy()).cuda()
            ids, sc = search_local_shards(ss, dq, p, N)
            eids, esc, tr = port.search(whole, q, p)
            assert np.array_equal(ids, eids), (G, p)
            assert np.array_equal(bits(sc), bits(esc)), (G, p)
            c = torch.zeros(6, dtype=torch.int64, device="cuda")
            tot = np.zeros(6, np.int64)
            for s in ss:
                s.trace_counters_device(c.data_ptr())
                torch.cuda.synchronize()
                tot += c.cpu().numpy()
            assert tot[0] == tr["stage1_candidates"] and tot[1] == tr["stage2_out"]
            assert tot[2] == tr["stage3_out"]
            assert tot[4] == tr["stage2_rows_gathered"] and tot[5] == tr["stage3_rows_gathered"]
    # disable_filter: nothing is cut before stage 4
    p = P.default_params_for_k(10)
    dq = torch.from_numpy(qs[0].copy()).cuda()
    ids, sc = search_local_shards(ss, dq, p, N, options=P.SearchOptions(disable_filter=True))
    eids, esc, _ = port.search(whole, qs[0], p, disable_filter=True)
    assert np.array_equal(ids, eids) and np.array_equal(bits(sc), bits(esc))


@pytest.mark.parametrize("lanes", [1, 3, 8])
def test_batch_searcher_bit_exact(small, port, lanes):
    """Throughput mode: every query of a batch spread over `lanes` concurrent
    streams returns exactly the reference's single-query result."""
    h, qs, idx, _ = small
    b = P.BatchSearcher(idx, lanes=lanes, score_mode=P.ScoreMode.EXACT, engine="lanes")
    qb = np.concatenate([qs, qs[::-1], qs[:3]])
    for k in (10, 1000):
        p = P.default_params_for_k(k)
        got = b.search(qb, p)
        assert len(got) == len(qb)
        for q, g in zip(qb, got):
            ids, sc, _ = port.search(h, q, p)
            assert np.array_equal(g.passage_ids, ids)
            assert np.array_equal(bits(g.scores), bits(sc))
    # one bad query rejects the whole batch before any work (types.cpp:61-72)
    bad = qb.copy()
    bad[2, 0, :] *= 2.0
    with pytest.raises(P.PlaidError):
        b.search(bad, P.default_params_for_k(10))


@pytest.mark.parametrize("lanes", [2, 5])
def test_batch_tensor_scores_match_single(small, lanes):
    """Batched S_cq (two queries per pass over C, N = 128 MMAs) gives the same
    results as the single-query tensor kernel, query by query; odd batch
    sizes end with a one-query pass."""
    h, qs, idx, _ = small
    single = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
    b = P.BatchSearcher(idx, lanes=lanes, score_mode=P.ScoreMode.TENSOR, engine="lanes")
    qb = np.concatenate([qs, qs[1:4]])  # 9 queries
    for k in (10, 100, 1000):
        p = P.default_params_for_k(k)
        got = b.search(qb, p)
        for q, g in zip(qb, got):
            r = single.search(q, p)
            assert np.array_equal(g.passage_ids, r.topk.passage_ids), k
            assert np.array_equal(bits(g.scores), bits(r.topk.scores)), k


def test_index_open_gpu_checksums(tmp_path, small, port):
    """On-disk index -> DeviceIndex.open (mmap, one upload, checksums verified
    on the GPU over the HBM copies) searches exactly like the in-memory index;
    a flipped byte is a ChecksumMismatch naming the file."""
    h, qs, idx, s = small
    P.save_index(h, tmp_path)
    ix2 = P.DeviceIndex.open(tmp_path, validate=True)
    s2 = P.Searcher(ix2)
    p = P.default_params_for_k(100)
    for q in qs[:3]:
        a, b = s.search(q, p), s2.search(q, p)
        assert np.array_equal(a.topk.passage_ids, b.topk.passage_ids)
        assert np.array_equal(bits(a.topk.scores), bits(b.topk.scores))
    f = tmp_path / "codes.u32"
    raw = bytearray(f.read_bytes())
    raw[123] ^= 0x10
    f.write_bytes(bytes(raw))
    with pytest.raises(P.PlaidError) as e:
        P.DeviceIndex.open(tmp_path)
    assert e.value.code == P.ErrorCode.ChecksumMismatch and "codes.u32" in str(e.value)
    (tmp_path / "doclens.u32").write_bytes(b"\0" * 8)
    with pytest.raises(P.PlaidError) as e:
        P.DeviceIndex.open(tmp_path)
    assert e.value.code == P.ErrorCode.LengthMismatch


def test_graph_replay_matches_eager(small, port):
    """use_graphs: the host path captured as one CUDA graph per (rows, params)
    and replayed returns exactly the eager results; growing k re-allocates
    the result block, so the cached graphs are re-captured."""
    h, qs, idx, s = small
    g = P.Searcher(idx, score_mode=P.ScoreMode.EXACT, use_graphs=True)
    for k in (10, 100, 10, 1000, 100):
        p = P.default_params_for_k(k)
        for q in qs:
            a, b = s.search(q, p), g.search(q, p)
            assert np.array_equal(a.topk.passage_ids, b.topk.passage_ids), k
            assert np.array_equal(bits(a.topk.scores), bits(b.topk.scores)), k
            assert a.trace.counters() == b.trace.counters()
        ids, sc, _ = port.search(h, qs[0], p)
        assert np.array_equal(g.search(qs[0], p).topk.passage_ids, ids)


@pytest.mark.parametrize("dim,nbits,K", [(64, 2, 96), (128, 1, 300), (32, 4, 17)])
def test_encode_matches_reference_build(dim, nbits, K):
    """GPU encode (assign_codes, quantise + pack, build_inverted_list) of a
    corpus against the centroids and quantizer the reference's build_index
    trained on it: codes, residual bytes and the IVF are bit-identical."""
    import oracle

    if not oracle.available("ref"):
        pytest.skip("compiled reference not available")
    ref = oracle.get("ref")
    rng = np.random.default_rng(dim + K)
    doclens = rng.integers(1, 40, 250).astype(np.uint32)
    x = rng.standard_normal((int(doclens.sum()), dim)).astype(np.float32)
    x /= np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True).astype(np.float32)
    x = (x / np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
    d = ref.build_index(x, doclens, dim, nbits, K, iters=3, seed=5)
    h = P.encode_corpus(x, doclens, d["centroids"], d["bucket_cutoffs"], d["bucket_weights"], nbits)
    assert np.array_equal(h.codes, d["codes"])
    assert np.array_equal(h.residuals, d["residuals"])
    assert np.array_equal(h.ivf_offsets, d["ivf_offsets"])
    assert np.array_equal(h.ivf_postings, d["ivf_postings"])
    # and the encoded index searches like the reference-built one
    port = oracle.get("port")
    hr = P.HostIndex(dim, nbits, d["centroids"], d["codes"], d["residuals"], d["doclens"], d["ivf_offsets"],
                     d["ivf_postings"], d["bucket_cutoffs"], d["bucket_weights"])
    q = x[:32] if dim >= 32 else x[:32]
    s = P.Searcher(P.DeviceIndex.from_host(h), score_mode=P.ScoreMode.EXACT)
    p = P.SearchParams(10, 2, 0.3, 64)
    got = s.search(q, p)
    ids, sc, _ = port.search(hr, q, p)
    assert np.array_equal(got.topk.passage_ids, ids)


def test_encode_rejects_bad_corpus():
    x = np.ones((4, 8), np.float32)
    with pytest.raises(P.PlaidError) as e:
        P.encode_corpus(x, np.array([2, 2], np.uint32), np.eye(8, dtype=np.float32)[:2], np.zeros(3, np.float32),
                        np.zeros(4, np.float32), 2)
    assert e.value.code == P.ErrorCode.NotNormalized


@pytest.mark.parametrize("K", [300, 129, 33])
def test_partial_last_tile(port, K):
    """K not a multiple of the S_cq tile (128 centroids, 32 per lane group):
    both score modes must ignore the rows past K (regression: an unsigned
    underflow let the last tile write S rows and candidate ids beyond K)."""
    h = P.generate_index(1500, K, dim=128, nbits=2, mean_len=30, seed=K)
    qs = P.generate_queries(h, 3, seed=1)
    idx = P.DeviceIndex.from_host(h)
    for mode in (P.ScoreMode.EXACT, P.ScoreMode.TENSOR):
        s = P.Searcher(idx, score_mode=mode)
        for q in qs:
            S, mx = s.compute_centroid_scores(q)
            S0, mx0 = port.compute_centroid_scores(h, q)
            assert np.abs(S - S0).max() < 5e-6
            got = s.search(q, P.default_params_for_k(10))
            if mode == P.ScoreMode.EXACT:
                ids, sc, _ = port.search(h, q, P.default_params_for_k(10))
                assert np.array_equal(got.topk.passage_ids, ids)
            assert np.all(got.topk.passage_ids < h.num_passages)


def test_edge_cases(port):
    """Empty stage-1 candidate set (pipeline.cpp:249-252: empty result), the
    generic nprobe > 32 path, short queries (|Q| < 32), k above the corpus."""
    rng = np.random.default_rng(3)
    base = P.generate_index(400, 64, dim=64, nbits=2, mean_len=12, spread=4, seed=8)
    # move every token onto centroids 0..31: centroids 32..63 own no passages
    codes = (base.codes % 32).astype(np.uint32)
    ivf_off, post = P.build_inverted_list(codes, base.doclens, 64)
    h = P.HostIndex(base.dim, base.nbits, base.centroids, codes, base.residuals, base.doclens, ivf_off, post,
                    base.bucket_cutoffs, base.bucket_weights)
    s = P.Searcher(P.DeviceIndex.from_host(h), score_mode=P.ScoreMode.EXACT)
    q = np.repeat(h.centroids[63:64], 4, axis=0)  # its only top-1 centroid is empty
    for p in (P.SearchParams(10, 1, 0.5, 64), P.SearchParams(5, 1, -1.0, 64)):
        got = s.search(q, p)
        ids, sc, tr = port.search(h, q, p)
        assert len(got.topk) == 0 == len(ids) and got.trace.counters() == tr
    qs = P.generate_queries(h, 3, seed=4)
    for rows in (1, 8, 32):
        for p in (P.SearchParams(10, 40, 0.4, 256), P.SearchParams(500, 6, 0.3, 2000), P.SearchParams(3, 63, 0.5, 12)):
            for q in qs:
                qq = q[:rows] if rows < 32 else q
                got = s.search(qq, p)
                ids, sc, tr = port.search(h, qq, p)
                assert np.array_equal(got.topk.passage_ids, ids), (rows, p)
                assert np.array_equal(bits(got.topk.scores), bits(sc))
                assert got.trace.counters() == tr


def test_merge_topk_rows_device(port):
    """Packed per-shard rows [k pids | k scores | u64 count] (one all-gather
    per query) merge like the separate arrays."""
    import torch

    rng = np.random.default_rng(9)
    s = P.Searcher(None)
    G, k = 5, 64
    counts = [64, 10, 0, 64, 33]
    rows = np.zeros((G, 2 * k + 2), np.uint32)
    allp, alls = [], []
    for g in range(G):
        c = counts[g]
        p = (rng.permutation(5000)[:c] + g * 5000).astype(np.uint32)
        v = np.sort(rng.standard_normal(c).astype(np.float32))[::-1].copy()
        rows[g, :c] = p
        rows[g, k:k + c] = v.view(np.uint32)
        rows[g, 2 * k:].view(np.uint64)[0] = c
        allp.append(p), alls.append(v)
    d = torch.from_numpy(rows.reshape(-1).view(np.int32)).cuda()
    op = torch.zeros(k, dtype=torch.int32, device="cuda")
    os_ = torch.zeros(k, dtype=torch.float32, device="cuda")
    on = torch.zeros(1, dtype=torch.int64, device="cuda")
    s.merge_topk_rows_device(d.data_ptr(), G, k, op.data_ptr(), os_.data_ptr(), on.data_ptr())
    torch.cuda.synchronize()
    b = port.select_top(np.concatenate(allp), np.concatenate(alls), k)
    m = int(on[0])
    assert np.array_equal(op[:m].cpu().numpy().view(np.uint32), b[0])
    assert np.array_equal(os_[:m].cpu().numpy(), b[1])


@pytest.mark.gpu
def test_batch_sharded_global_exact_world1(port):
    """Global-exact throughput mode (sharded.BatchShardedSearcher) on one GPU
    in a world-size-1 NCCL group: 7 queries through 3 lane Searchers (a
    ragged last wave), each lane on its own stream, the exchanges and
    rank-major transposes on the caller's stream.  Every [b][k] row equals
    the reference search of query b, bit for bit."""
    import socket

    import torch
    import torch.distributed as dist

    from paper_2205_09707_b200.sharded import BatchShardedSearcher

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port_no = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_no))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        N, K = 6000, 512
        h = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
        qs = P.generate_queries(h, 7, seed=21)
        ix = P.DeviceIndex.from_host_at(h, pid_base=0)
        for p in [P.default_params_for_k(10), P.default_params_for_k(100), P.SearchParams(50, 4, 0.3, 64)]:
            lanes = [P.Searcher(ix, score_mode=P.ScoreMode.EXACT, record_times=False) for _ in range(3)]
            bs = BatchShardedSearcher(lanes, k=p.k, num_passages=N, device=torch.device("cuda", 0))
            dq = torch.from_numpy(np.ascontiguousarray(qs)).cuda()
            op = torch.zeros(len(qs), p.k, dtype=torch.int32, device="cuda")
            osc = torch.zeros(len(qs), p.k, dtype=torch.float32, device="cuda")
            on = torch.zeros(len(qs), dtype=torch.int64, device="cuda")
            bs.search(dq, p, op, osc, on)
            torch.cuda.synchronize()
            assert bs.launches > 0
            for b, q in enumerate(qs):
                ids, sc, _ = port.search(h, q, p)
                m = int(on[b])
                assert np.array_equal(op[b, :m].cpu().numpy().view(np.uint32), ids), (p, b)
                assert np.array_equal(bits(osc[b, :m].cpu().numpy()), bits(sc)), (p, b)
    finally:
        dist.destroy_process_group()

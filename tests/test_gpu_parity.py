"""GPU parity: the CUDA engine (through the C ABI) against the CPU oracle on
identical index bytes and queries.  Integer outputs and, in EXACT score mode,
every fp32 score must be bit-identical to the reference arithmetic."""
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

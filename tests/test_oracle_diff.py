"""The C restatement (oracle/plaid_oracle.c) against the compiled reference
(oracle/_ref, built from /root/reference/proj/src) on identical index bytes
and queries: every integer output and every fp32 score bit must agree.  Also
the SPEC acceptance properties that involve the whole pipeline (#1, #6, #7)
and the stage-trace invariants."""
import numpy as np
import pytest

import oracle
import paper_2205_09707_b200 as P

pytestmark = pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module", params=[(128, 2, 0), (64, 1, 1), (16, 4, 2), (128, 1, 3)],
                ids=["d128b2", "d64b1", "d16b4", "d128b1"])
def case(request):
    dim, nbits, seed = request.param
    h = P.generate_index(600, 64, dim=dim, nbits=nbits, mean_len=24, spread=8, seed=seed)
    qs = P.generate_queries(h, 3, seed=100 + seed)
    return h, qs


def test_index_validates(case, ref):
    ref.validate_index(case[0])


@pytest.mark.parametrize("k", [1, 10, 100, 1000])
def test_search_port_equals_ref(case, port, ref, k):
    h, qs = case
    p = P.default_params_for_k(k)
    for q in qs:
        a = port.search(h, q, p)
        b = ref.search(h, q, p, threads=2)
        assert np.array_equal(a[0], b[0])
        assert np.array_equal(bits(a[1]), bits(b[1]))
        assert a[2] == b[2]


@pytest.mark.parametrize("params", [(10, 3, 0.3, 64), (50, 64, -1.0, 2400), (7, 2, 0.9, 16), (20, 5, 0.45, 20)])
def test_search_params_sweep(case, port, ref, params):
    h, qs = case
    p = P.SearchParams(*params)
    for disable in (False, True):
        a = port.search(h, qs[0], p, disable_filter=disable)
        b = ref.search(h, qs[0], p, disable_filter=disable, threads=1)
        assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1])) and a[2] == b[2]


def test_stages_port_equals_ref(case, port, ref):
    h, qs = case
    q = qs[1]
    S, mx = port.compute_centroid_scores(h, q)
    S2, mx2 = ref.compute_centroid_scores(h, q)
    assert np.array_equal(bits(S), bits(S2)) and np.array_equal(bits(mx), bits(mx2))
    for nprobe in (1, 2, 5, h.num_centroids):
        assert np.array_equal(port.generate_candidates(h, S, nprobe), ref.generate_candidates(h, S, nprobe))
    c1 = port.generate_candidates(h, S, 4)
    for t_cs in (-1.0, 0.3, 0.5):
        keep = port.prune_centroids(mx, t_cs)
        assert np.array_equal(keep, ref.prune_centroids(mx, t_cs))
        a = port.centroid_interaction(h, c1, S, keep)
        b = ref.centroid_interaction(h, c1, S, keep)
        assert np.array_equal(bits(a[0]), bits(b[0])) and a[1] == b[1]
    a = port.centroid_interaction(h, c1, S, None)
    b = ref.centroid_interaction(h, c1, S, None)
    assert np.array_equal(bits(a[0]), bits(b[0])) and a[1] == b[1]
    for n in (1, 17, len(c1), len(c1) + 3):
        x, y = port.select_top(c1, a[0], n), ref.select_top(c1, a[0], n)
        assert np.array_equal(x[0], y[0]) and np.array_equal(bits(x[1]), bits(y[1]))
    x, y = port.rank_final(h, c1[:50], q, 20), ref.rank_final(h, c1[:50], q, 20)
    assert np.array_equal(x[0], y[0]) and np.array_equal(bits(x[1]), bits(y[1]))
    codes = h.codes[:200]
    res = h.residuals[: 200 * h.bytes_per_token]
    assert np.array_equal(bits(port.reconstruct(h, codes, res)), bits(ref.reconstruct(h, codes, res)))


def test_acceptance1_exhaustive_equivalence(case, port, ref):
    """nprobe=K, t_cs=-1, ndocs=4N reproduces the exhaustive
    decompressed-Eq.1 top-k (ids and order exact)."""
    h, qs = case
    allp = np.arange(h.num_passages, dtype=np.uint32)
    p = P.SearchParams(25, h.num_centroids, -1.0, 4 * h.num_passages)
    for q in qs:
        ids, sc, tr = ref.search(h, q, p, threads=2)
        ex_ids, ex_sc = ref.rank_final(h, allp, q, 25)
        assert np.array_equal(ids, ex_ids) and np.array_equal(bits(sc), bits(ex_sc))
        # Eq. 1 in float64 from the reconstructed embeddings, within 1e-5
        emb = ref.reconstruct(h, h.codes, h.residuals).astype(np.float64)
        for pid, s in zip(ids[:5], sc[:5]):
            a, b = h.passage_offsets[pid], h.passage_offsets[pid + 1]
            eq1 = (q.astype(np.float64) @ emb[a:b].T).max(axis=1).sum()
            assert abs(eq1 - s) < 1e-5


def test_acceptance6_pruning_consistency(case, port):
    """at t_cs=-1 stage-2 scores equal stage-3 scores; raising
    t_cs never increases the gathered-row count."""
    h, qs = case
    S, mx = port.compute_centroid_scores(h, qs[0])
    c1 = port.generate_candidates(h, S, 3)
    s2, r2 = port.centroid_interaction(h, c1, S, port.prune_centroids(mx, -1.0))
    s3, r3 = port.centroid_interaction(h, c1, S, None)
    assert np.array_equal(bits(s2), bits(s3)) and r2 == r3
    rows = [port.centroid_interaction(h, c1, S, port.prune_centroids(mx, t))[1]
            for t in (-1.0, 0.0, 0.2, 0.4, 0.6, 0.8, 1.0)]
    assert all(a >= b for a, b in zip(rows, rows[1:]))


def test_acceptance7_and_trace_monotone(case, port):
    """SPEC.md:615 + :387: decompressed passages = min(ceil(ndocs/4) or k,
    stage-3 input); stage1 >= stage2_out >= stage3_out >= |result|."""
    h, qs = case
    for k in (1, 10, 100):
        p = P.default_params_for_k(k)
        ids, sc, tr = port.search(h, qs[2], p)
        w = P.stage3_width(p)
        assert tr["stage2_out"] == min(p.ndocs, tr["stage1_candidates"])
        assert tr["stage3_out"] == min(w, tr["stage2_out"])
        assert tr["decompressed_passages"] == tr["stage3_out"]
        assert tr["final_out"] == len(ids) == min(k, tr["stage3_out"])
        assert tr["centroid_matmul_count"] == 1
        assert np.all(np.diff(sc) <= 0)


def test_determinism(case, port, ref):
    h, qs = case
    p = P.default_params_for_k(10)
    a = ref.search(h, qs[0], p, threads=1)
    b = ref.search(h, qs[0], p, threads=8)
    c = port.search(h, qs[0], p)
    assert np.array_equal(a[0], b[0]) and np.array_equal(bits(a[1]), bits(b[1]))
    assert np.array_equal(a[0], c[0]) and np.array_equal(bits(a[1]), bits(c[1]))

"""Throughput mode, wave engine (csrc/wave_scores.cu, csrc/wave_worker.cu):
one S_cq pass per wave of queries and one CTA per query for stages 1b-4.

EXACT score mode runs the exact S_cq per query, and everything after S is the
reference's arithmetic, so every result, score bit and StageTrace counter
equals lir::search (pipeline.cpp:232-283; the oracle pinned to it).  TENSOR
mode (four queries per tcgen05 pass over C) is classified with the north_star
comparator (oracle/compare.py) against the S table the wave actually used.
"""
import numpy as np
import pytest

import paper_2205_09707_b200 as P
from oracle.compare import check_tensor_search

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


@pytest.fixture(scope="module")
def idx_small():
    h = P.generate_index(20000, 1024, dim=128, nbits=2, mean_len=48, seed=5)
    qs = P.generate_queries(h, 13, seed=21)
    return h, qs, P.DeviceIndex.from_host(h)


@pytest.fixture(scope="module")
def idx_nb1():
    # cfg3-shaped (nbits = 1) at test scale; K not a multiple of 128 (partial last tile)
    h = P.generate_index(12000, 1000, dim=128, nbits=1, mean_len=68, seed=9)
    qs = P.generate_queries(h, 9, seed=4)
    return h, qs, P.DeviceIndex.from_host(h)


def _counters(tr):
    return [tr["stage1_candidates"], tr["stage2_out"], tr["stage3_out"], tr["final_out"]]


@pytest.mark.parametrize("k", [1, 10, 100, 1000])
def test_wave_exact_bit_exact(idx_small, port, k):
    h, qs, idx = idx_small
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT)
    p = P.default_params_for_k(k)
    res = b.search(qs, p)
    assert b.last_was_wave()
    cnt = b.counters(len(qs))
    for j, q in enumerate(qs):
        ids, sc, tr = port.search(h, q, p)
        assert np.array_equal(res[j].passage_ids, ids), j
        assert np.array_equal(bits(res[j].scores), bits(sc)), j
        assert list(cnt[j]) == _counters(tr), (j, list(cnt[j]), tr)


@pytest.mark.parametrize("k", [10, 100])
def test_wave_exact_nbits1_partial_tile(idx_nb1, port, k):
    h, qs, idx = idx_nb1
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT)
    p = P.default_params_for_k(k)
    res = b.search(qs, p)
    assert b.last_was_wave()
    cnt = b.counters(len(qs))
    for j, q in enumerate(qs):
        ids, sc, tr = port.search(h, q, p)
        assert np.array_equal(res[j].passage_ids, ids), j
        assert np.array_equal(bits(res[j].scores), bits(sc)), j
        assert list(cnt[j]) == _counters(tr), j


@pytest.mark.parametrize("t_cs", [-1.0, 0.2, 0.45, 0.9])
def test_wave_exact_t_cs_paths(idx_small, port, t_cs):
    """t_cs near -1 keeps every centroid: stage 2 scans codes instead of
    walking posting lists; t_cs = 0.9 keeps almost nothing (zero-score
    boundary bucket in the radix select)."""
    h, qs, idx = idx_small
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT)
    p = P.SearchParams(k=50, nprobe=3, t_cs=t_cs, ndocs=400)
    res = b.search(qs[:5], p)
    assert b.last_was_wave()
    for j, q in enumerate(qs[:5]):
        ids, sc, tr = port.search(h, q, p)
        assert np.array_equal(res[j].passage_ids, ids), j
        assert np.array_equal(bits(res[j].scores), bits(sc)), j


def test_wave_matches_lanes(idx_small):
    h, qs, idx = idx_small
    p = P.default_params_for_k(100)
    a = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT).search(qs, p)
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT, engine="lanes").search(qs, p)
    for x, y in zip(a, b):
        assert np.array_equal(x.passage_ids, y.passage_ids) and np.array_equal(bits(x.scores), bits(y.scores))


@pytest.mark.parametrize("k", [10, 100, 1000])
def test_wave_tensor_comparator(idx_small, ref, k):
    """Four queries per tcgen05 pass (13 queries: a partial last group)."""
    h, qs, idx = idx_small
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.TENSOR)
    p = P.default_params_for_k(k)
    res = b.search(qs, p)
    assert b.last_was_wave()
    cnt = b.counters(len(qs))
    rows = qs.shape[1]
    for j, q in enumerate(qs):
        S = b.wave_scores(j)[:, :rows]
        got = dict(zip(("stage1_candidates", "stage2_out", "stage3_out", "final_out"), (int(x) for x in cnt[j])))
        rep = check_tensor_search(ref, h, q, p, res[j].passage_ids, res[j].scores, S, got_counters=got)
        assert rep.ok, (j, rep.problems)
        # stage 4 on mma.sync: (S + R Q^T) * inv with a three-way bf16 split of
        # the residual product (~1e-6 relative observed; north_star allows 1e-4)
        assert rep.max_rel_score_err < 2e-5


def test_wave_tensor_many_tiles_per_cta(port):
    """K = 2^16 at 148 CTAs: ~3.5 tiles per CTA per group, several groups, the
    8-box ring wraps many times, both accumulators and the A reload run."""
    h = P.generate_index(30000, 1 << 16, dim=128, nbits=2, mean_len=32, seed=12)
    qs = P.generate_queries(h, 10, seed=3)
    idx = P.DeviceIndex.from_host(h)
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.TENSOR)
    p = P.default_params_for_k(10)
    b.search(qs, p)
    assert b.last_was_wave()
    rows = qs.shape[1]
    for j, q in enumerate(qs):
        S = b.wave_scores(j)[:, :rows]
        S0, _ = port.compute_centroid_scores(h, q)
        assert np.abs(S - S0).max() < 5e-6, j


def test_wave_rejects_bad_query_on_device(idx_small):
    h, qs, idx = idx_small
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.TENSOR)
    import torch

    q = torch.tensor(qs, device="cuda")
    q[3, 0, :] *= 2.0
    nq, rows, dim = q.shape
    p = P.default_params_for_k(10)
    pids = torch.zeros(nq * 10, dtype=torch.int32, device="cuda")
    sc = torch.zeros(nq * 10, dtype=torch.float32, device="cuda")
    n = torch.zeros(nq, dtype=torch.int64, device="cuda")
    b.search_device(q.data_ptr(), nq, rows, dim, p, pids.data_ptr(), sc.data_ptr(), n.data_ptr())
    with pytest.raises(P.PlaidError) as e:
        b.sync()
    assert e.value.code == P.ErrorCode.NotNormalized


def test_wave_more_queries_than_slots(idx_nb1, port):
    """A batch larger than the wave runs in several waves (slot reuse: the
    bitmap and accumulators are left clean for the next query)."""
    h, qs, idx = idx_nb1
    big = np.concatenate([qs] * 80)  # 720 queries > 512 slots
    b = P.BatchSearcher(idx, score_mode=P.ScoreMode.EXACT)
    p = P.default_params_for_k(10)
    res = b.search(big, p)
    assert b.last_was_wave()
    for j in (0, 5, 511, 512, 600, 719):
        ids, sc, _ = port.search(h, big[j], p)
        assert np.array_equal(res[j].passage_ids, ids), j
        assert np.array_equal(bits(res[j].scores), bits(sc)), j

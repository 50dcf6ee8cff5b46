"""SPEC.md acceptance properties checked on the B200 engine itself (the CPU
suite checks them on the oracle): #5 self-recall curve, #6 pruning
consistency, #7 pipeline-work bound, #9 latency shape (
paper §3.2-§3.4)."""
import math

import numpy as np
import pytest

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import analysis

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mid():
    h = P.generate_index(3000, 256, dim=64, nbits=2, mean_len=24, spread=8, seed=12)
    qs = P.generate_queries(h, 4, seed=5)
    return h, qs, P.Searcher(P.DeviceIndex.from_host(h), score_mode=P.ScoreMode.EXACT)


def test_self_recall_curve(mid):
    """#5: recall of the exhaustive top-k inside the centroid-only top-k' is
    monotone non-decreasing in k' and reaches 1 at k' = N."""
    h, qs, s = mid
    rows = analysis.self_recall(s, qs[:3], ks=(10, 100), kprimes=(10, 50, 100, 500, 1000, 3000))
    for k in (10, 100):
        curve = [r for kk, kp, r in rows if kk == k]
        assert all(b >= a - 1e-12 for a, b in zip(curve, curve[1:])), curve
        assert curve[-1] == pytest.approx(1.0)
    # the query's source passage shapes the head: top-10 within top-100 is high
    assert [r for kk, kp, r in rows if kk == 10 and kp == 100][0] >= 0.5


def test_pruning_consistency(mid, port):
    """#6: with t_cs = -1 (nothing pruned) stage-2 and stage-3 scores agree for
    every candidate; raising t_cs never increases the stage-2 rows gathered."""
    h, qs, s = mid
    q = qs[0]
    S, mx = s.compute_centroid_scores(q)
    c1 = s.generate_candidates(S, 8)
    keep = s.prune_centroids(mx, -1.0)
    a, ra = s.centroid_interaction(c1, S, keep)
    b, rb = s.centroid_interaction(c1, S, None)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32)) and ra == rb
    rows = []
    for t_cs in (-1.0, 0.0, 0.2, 0.3, 0.4, 0.5, 0.7, 1.0):
        rows.append(s.search(q, P.SearchParams(10, 8, t_cs, 256)).trace.stage2_rows_gathered)
    assert all(y <= x for x, y in zip(rows, rows[1:])), rows


@pytest.mark.parametrize("ndocs", [16, 64, 256, 1024])
def test_pipeline_work_bound(mid, ndocs):
    """#7: fully decompressed passages = min(ceil(ndocs / 4), |stage-3 input|)
    (k <= ndocs / 4, so stage3_width = ceil(ndocs / 4), pipeline.cpp:227-230)."""
    h, qs, s = mid
    for q in qs:
        tr = s.search(q, P.SearchParams(4, 2, 0.4, ndocs)).trace
        assert tr.decompressed_passages == min(math.ceil(ndocs / 4), tr.stage2_out)


def test_filter_latency_shape():
    """#9 analog: stages 2-3 cut the stage-4 (lookup + decompression + scoring)
    time by >= 3x against disable_filter, which decompresses every stage-1
    candidate; with ndocs covering every candidate the top-k are identical."""
    h = P.generate_index(100_000, 4096, dim=128, nbits=2, mean_len=64, spread=16, seed=3)
    qs = P.generate_queries(h, 5, seed=9)
    s = P.Searcher(P.DeviceIndex.from_host(h), score_mode=P.ScoreMode.EXACT, record_times=True)
    r = analysis.filter_speedup(s, qs, P.default_params_for_k(10))
    assert r["speedup"] >= 3.0, r
    wide = P.SearchParams(10, 2, -1.0, 4 * h.num_passages)
    for q in qs[:2]:
        a = s.search(q, wide)
        b = s.search(q, wide, P.SearchOptions(disable_filter=True))
        assert np.array_equal(a.topk.passage_ids, b.topk.passage_ids)


def test_centroid_score_cdf(mid):
    h, qs, s = mid
    v, cdf = analysis.centroid_score_cdf(s, qs[0])
    assert v.size == h.num_centroids and np.all(np.diff(v) >= 0) and cdf[-1] == 1.0
    S, mx = s.compute_centroid_scores(qs[0])
    assert np.array_equal(np.sort(S.max(axis=1)), v)

"""The paper's desk-scale analyses on the B200 engine (
SPEC.md cli-bench "cmd_selfrecall" / "cmd_centroid_cdf", acceptance #5, #6,
#9).  Everything runs through the engine's own per-stage entry points.

* self_recall — §3.3 / Fig. 3: the fraction of the exhaustive (decompressed,
  exact MaxSim over every passage) top-k found inside the centroid-only
  (stage-3 score, no residuals) top-k'.
* centroid_score_cdf — §3.4 / Fig. 3: the empirical CDF of every centroid's
  maximum score over the query tokens.
* filter_speedup — §3.2 / Fig. 2 analog: stage-4 (lookup + decompression +
  scoring) time with stages 2-3 enabled versus `disable_filter`, which sends
  every stage-1 candidate to stage 4.
"""
from __future__ import annotations

import numpy as np

from .api import SearchOptions, SearchParams, Searcher


def exhaustive_topk(s: Searcher, q: np.ndarray, k: int) -> np.ndarray:
    """Exact Eq.-1 top-k over every passage (decompress + MaxSim on the GPU)."""
    n = s.index.num_passages
    ids, _ = s.rank_final(np.arange(n, dtype=np.uint32), q, min(k, n))
    return ids


def centroid_only_ranking(s: Searcher, q: np.ndarray, kmax: int) -> np.ndarray:
    """Passages ranked by the unmasked centroid interaction (stage 3's score)."""
    n = s.index.num_passages
    S, _ = s.compute_centroid_scores(q)
    allp = np.arange(n, dtype=np.uint32)
    sc, _ = s.centroid_interaction(allp, S, None)
    ids, _ = s.select_top(allp, sc, min(kmax, n))
    return ids


def self_recall(s: Searcher, queries: np.ndarray, ks=(10, 100, 1000), kprimes=(10, 20, 50, 100, 200, 500, 1000,
                                                                                 2000)) -> list[tuple[int, int, float]]:
    """Rows (k, k', mean recall over the queries) for k <= N and k' >= k."""
    n = s.index.num_passages
    ks = [k for k in ks if k <= n]
    kps = sorted({min(kp, n) for kp in kprimes})
    out = []
    for k in ks:
        rec = np.zeros(len(kps))
        for q in queries:
            truth = set(exhaustive_topk(s, q, k).tolist())
            ranked = centroid_only_ranking(s, q, max(kps))
            for j, kp in enumerate(kps):
                rec[j] += len(truth & set(ranked[:kp].tolist())) / len(truth)
        out += [(k, kp, float(r / len(queries))) for kp, r in zip(kps, rec) if kp >= k]
    return out


def centroid_score_cdf(s: Searcher, q: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """(sorted per-centroid max scores, CDF values i / K)."""
    _, mx = s.compute_centroid_scores(q)
    v = np.sort(mx)
    return v, np.arange(1, v.size + 1, dtype=np.float64) / v.size


def filter_speedup(s: Searcher, queries: np.ndarray, params: SearchParams) -> dict:
    """Stage-4 time (ms, mean over the queries) with and without stages 2-3
    and whether the top-k agree.  `s` must record phase times."""
    on, off, same = [], [], 0
    s.search(queries[0], params)  # warm-up: buffers sized, kernels configured
    s.search(queries[0], params, SearchOptions(disable_filter=True))
    for q in queries:
        a = s.search(q, params)
        on.append(a.trace.decompression_ms)
        b = s.search(q, params, SearchOptions(disable_filter=True))
        off.append(b.trace.decompression_ms)
        same += int(np.array_equal(a.topk.passage_ids, b.topk.passage_ids))
    return {"stage4_ms_filtered": float(np.mean(on)), "stage4_ms_unfiltered": float(np.mean(off)),
            "speedup": float(np.mean(off) / max(np.mean(on), 1e-9)), "identical_topk": same / len(queries)}

"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run here (where /root/reference exists and oracle/_ref/liblir_ref.so is
built by `make -C oracle ref`):

    python tests/golden/make_golden.py

For each case a clustered random corpus is indexed by the reference's own
offline builder (lir::build_index: k-means, assign, quantise, pack, IVF —
indexer.cpp:197-282), and the reference's `lir::search` (pipeline.cpp:232-283)
and per-stage functions are run on seeded queries.  The fixture stores the
index arrays, the queries, and every expected output (ids, score BITS, stage
traces, S_cq bits, C1, keep mask, stage-2 scores).  Nothing here runs on the
GPU box; the fixtures travel as committed files.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import oracle  # noqa: E402
from paper_2205_09707_b200.hostindex import HostIndex  # noqa: E402

OUT = Path(__file__).resolve().parent
# (name, dim, nbits, K, N, mean_len, seed)
CASES = [("d128_b2", 128, 2, 32, 120, 20, 1), ("d64_b1", 64, 1, 16, 80, 12, 2), ("d32_b4", 32, 4, 16, 60, 10, 3)]
PARAMS = [(1, 1, 0.5, 256), (10, 1, 0.5, 256), (10, 2, 0.3, 40), (100, 2, 0.45, 1024), (1000, 4, 0.4, 4096),
          (5, 16, -1.0, 1000)]


class Prm:
    def __init__(self, k, nprobe, t_cs, ndocs):
        self.k, self.nprobe, self.t_cs, self.ndocs = k, nprobe, t_cs, ndocs


def corpus(dim, N, mean_len, seed):
    rng = np.random.default_rng(seed)
    topics = rng.standard_normal((12, dim))
    doclens = rng.integers(max(1, mean_len - 6), mean_len + 7, size=N).astype(np.uint32)
    rows = []
    for p in range(N):
        t = topics[rng.integers(0, 12, size=3)]
        x = t[rng.integers(0, 3, size=int(doclens[p]))] + 0.6 * rng.standard_normal((int(doclens[p]), dim))
        rows.append(x)
    data = np.concatenate(rows).astype(np.float32)
    data /= np.linalg.norm(data, axis=1, keepdims=True)
    return data, doclens


def main():
    ref = oracle.get("ref")
    for name, dim, nbits, K, N, mean_len, seed in CASES:
        data, doclens = corpus(dim, N, mean_len, seed)
        d = ref.build_index(data, doclens, dim, nbits, K, iters=4, seed=seed, threads=1)
        h = HostIndex(d["dim"], d["nbits"], d["centroids"], d["codes"], d["residuals"], d["doclens"],
                      d["ivf_offsets"], d["ivf_postings"], d["bucket_cutoffs"], d["bucket_weights"])
        ref.validate_index(h)
        rng = np.random.default_rng(100 + seed)
        qs = []
        for _ in range(3):
            tok = data[rng.integers(0, data.shape[0], size=32)] + 0.05 * rng.standard_normal((32, dim))
            qs.append(tok / np.linalg.norm(tok, axis=1, keepdims=True))
        qs = np.stack(qs).astype(np.float32)
        fx = dict(d)
        fx["queries"] = qs
        fx["params"] = np.array([p[:2] + p[3:] for p in PARAMS], dtype=np.uint64)
        fx["params_tcs"] = np.array([p[2] for p in PARAMS], dtype=np.float32)
        for qi, q in enumerate(qs):
            for pi, p in enumerate(PARAMS):
                ids, sc, tr = ref.search(h, q, Prm(*p), threads=1)
                fx[f"ids_{qi}_{pi}"] = ids
                fx[f"scorebits_{qi}_{pi}"] = sc.view(np.uint32)
                fx[f"trace_{qi}_{pi}"] = np.array([tr[f] for f in sorted(tr)], dtype=np.uint64)
            S, mx = ref.compute_centroid_scores(h, q)
            c1 = ref.generate_candidates(h, S, 2)
            keep = ref.prune_centroids(mx, 0.45)
            s2, rows = ref.centroid_interaction(h, c1, S, keep)
            fx[f"Sbits_{qi}"] = S.view(np.uint32)
            fx[f"c1_{qi}"] = c1
            fx[f"keep_{qi}"] = keep
            fx[f"s2bits_{qi}"] = s2.view(np.uint32)
            fx[f"s2rows_{qi}"] = np.array([rows], dtype=np.uint64)
        fx["trace_fields"] = np.array(sorted(tr))
        np.savez_compressed(OUT / f"{name}.npz", **fx)
        print(f"{name}: K={K} N={N} T={h.num_embeddings} -> {OUT / (name + '.npz')}")


if __name__ == "__main__":
    main()

"""Throughput of the GPU encode (plaid_encode) on a synthetic corpus:
python tools/encode_bench.py [T_passages] [K] [dim] [nbits]"""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2205_09707_b200 as P  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 16
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 128
nbits = int(sys.argv[4]) if len(sys.argv) > 4 else 2
h = P.generate_index(N, K, dim=dim, nbits=nbits, mean_len=68, seed=0)
rng = np.random.default_rng(0)
x = rng.standard_normal((h.num_embeddings, dim)).astype(np.float32)
x = (x / np.linalg.norm(x.astype(np.float64), axis=1, keepdims=True)).astype(np.float32)
P.encode_corpus(x[:1000], np.array([1000], np.uint32), h.centroids, h.bucket_cutoffs, h.bucket_weights, nbits)
t = time.time()
e = P.encode_corpus(x, h.doclens, h.centroids, h.bucket_cutoffs, h.bucket_weights, nbits)
dt = time.time() - t
ops = 2.0 * h.num_embeddings * K * dim
print(f"T={h.num_embeddings} K={K} dim={dim}: {dt:.2f}s, {h.num_embeddings / dt / 1e6:.2f} M tokens/s, "
      f"assign {ops / dt / 1e12:.1f} T fp32 ops/s (incl. H2D/D2H), postings {len(e.ivf_postings)}")

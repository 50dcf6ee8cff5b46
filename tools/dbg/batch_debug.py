import sys; sys.path.insert(0, '.')
import numpy as np
import paper_2205_09707_b200 as P
K = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 16
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 1
h = P.generate_index(100000, K, dim=128, nbits=nb, mean_len=68, seed=0)
qs = P.generate_queries(h, 64, seed=3)
idx = P.DeviceIndex.from_host(h)
single = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
b = P.BatchSearcher(idx, lanes=8, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(100)
got = b.search(qs, p)
bad = 0
for q, g in zip(qs, got):
    r = single.search(q, p)
    bad += not np.array_equal(g.passage_ids, r.topk.passage_ids)
print("K", K, "mismatches", bad, "of", len(qs))

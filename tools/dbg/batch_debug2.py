import sys, os; sys.path.insert(0, '.')
import numpy as np
import paper_2205_09707_b200 as P
N = int(sys.argv[1]); nq = int(sys.argv[2]); L = int(sys.argv[3])
h = P.generate_index(N, 1 << 18, dim=128, nbits=1, mean_len=68, seed=0)
qs = P.generate_queries(h, nq, seed=3)
idx = P.DeviceIndex.from_host(h)
b = P.BatchSearcher(idx, lanes=L, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(100)
for it in range(3):
    got = b.search(qs, p)
print("ok", N, nq, L, len(got))

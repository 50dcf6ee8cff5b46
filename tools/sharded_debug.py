"""Debug: MultiGpuSearcher (C ABI plaid_sharded_*) global-exact vs the
unsharded oracle over several queries; prints every mismatch with trace."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200.sharded import shard_range  # noqa: E402

port = oracle.get("port")
G = int(sys.argv[1]) if len(sys.argv) > 1 else 3
N, K = 6000, 512
whole = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
qs = P.generate_queries(whole, 8, seed=21)
ixs = []
for g in range(G):
    a, b = shard_range(N, G, g)
    hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
    ixs.append(P.DeviceIndex.from_host_at(hs, pid_base=a))
ms = P.MultiGpuSearcher(ixs, score_mode=P.ScoreMode.EXACT)
bad = 0
for k in (10, 100, 1000):
    p = P.default_params_for_k(k)
    for qi, q in enumerate(qs):
        for rep in range(3):
            got = ms.search(q, p)
            ids, sc, tr = port.search(whole, q, p)
            c = got.trace.counters()
            if not (np.array_equal(got.topk.passage_ids, ids) and c == tr):
                bad += 1
                diff = {kk: (c[kk], tr[kk]) for kk in tr if c[kk] != tr[kk]}
                print(f"k={k} q={qi} rep={rep}: ids_equal={np.array_equal(got.topk.passage_ids, ids)} diff={diff}")
                gi, gs = got.topk.passage_ids, got.topk.scores
                print("  lens", len(gi), len(ids), "missing", sorted(set(ids.tolist()) - set(gi.tolist()))[:10],
                      "extra", sorted(set(gi.tolist()) - set(ids.tolist()))[:10])
                w = np.nonzero(gi[:min(len(gi), len(ids))] != ids[:min(len(gi), len(ids))])[0]
                for j in w[:6]:
                    print("   pos", j, "got", gi[j], gs[j], "exp", ids[j], sc[j])
                for j in np.nonzero(gs[:len(sc)] != sc[:len(gs)])[0][:4]:
                    print("   score pos", j, gs[j], sc[j])
print("mismatches", bad)

"""Stress the global-exact shard phases (tests/test_gpu_parity.py::
test_global_exact_shards_bit_exact) over many queries: summed per-shard trace
counters vs the unsharded oracle; prints every mismatch."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200.sharded import search_local_shards, shard_range  # noqa: E402

port = oracle.get("port")
G, N, K = 3, 6000, 512
whole = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
qs = P.generate_queries(whole, int(sys.argv[1]) if len(sys.argv) > 1 else 40, seed=21)
ss = []
for g in range(G):
    a, b = shard_range(N, G, g)
    hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
    ss.append(P.Searcher(P.DeviceIndex.from_host_at(hs, pid_base=a), score_mode=P.ScoreMode.EXACT))
bad = 0
for p in [P.default_params_for_k(10), P.default_params_for_k(100)]:
    for qi, q in enumerate(qs):
        dq = torch.from_numpy(q.copy()).cuda()
        ids, sc = search_local_shards(ss, dq, p, N)
        eids, esc, tr = port.search(whole, q, p)
        per = []
        for s in ss:
            c = torch.zeros(6, dtype=torch.int64, device="cuda")
            torch.cuda.synchronize()
            s.trace_counters_device(c.data_ptr())
            torch.cuda.synchronize()
            per.append(c.cpu().numpy())
        tot = np.sum(per, axis=0)
        ok = (np.array_equal(ids, eids) and tot[0] == tr["stage1_candidates"] and tot[1] == tr["stage2_out"]
              and tot[2] == tr["stage3_out"] and tot[4] == tr["stage2_rows_gathered"]
              and tot[5] == tr["stage3_rows_gathered"])
        if not ok:
            bad += 1
            print(f"MISMATCH k={p.k} q={qi}: per-shard {[x.tolist() for x in per]} oracle {tr} "
                  f"ids_equal={np.array_equal(ids, eids)}")
print(f"done: {bad} mismatches over {2 * len(qs)} searches")

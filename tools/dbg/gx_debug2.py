import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2205_09707_b200 as P
from paper_2205_09707_b200.sharded import shard_range, exchange_strides, search_local_shards
import oracle
port = oracle.get("port")
N, K, G = 6000, 512, 2
whole = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
qs = P.generate_queries(whole, 4, seed=21)
ss = []
for g in range(G):
    a, b = shard_range(N, G, g)
    hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
    ix = P.DeviceIndex.from_host_at(hs, pid_base=a)
    ss.append((ix, P.Searcher(ix, score_mode=P.ScoreMode.EXACT)))
c = torch.zeros(6, dtype=torch.int64, device="cuda")
def counters(s):
    s.trace_counters_device(c.data_ptr()); torch.cuda.synchronize(); return c.cpu().tolist()
for p in [P.default_params_for_k(k) for k in (10, 100)]:
    for qi, qq in enumerate(qs):
        q = torch.from_numpy(qq.copy()).cuda()
        ids, sc = search_local_shards([s for _, s in ss], q, p, N)
        ids0, sc0, tr = port.search(whole, qq, p)
        cs = [counters(s) for _, s in ss]
        print(p.k, qi, "match", np.array_equal(ids, ids0), cs, tr["stage1_candidates"], tr["stage2_out"], tr["stage3_out"])
        # rerun one shard alone (full search) to see its local counts
        for _, s in ss:
            r = s.search(qq, p)
            print("   local", r.trace.counters())

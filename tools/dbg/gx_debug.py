import sys; sys.path.insert(0, '.')
import numpy as np, torch
import paper_2205_09707_b200 as P
from paper_2205_09707_b200.sharded import shard_range, exchange_strides
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
p = P.default_params_for_k(10)
q = torch.from_numpy(qs[0].copy()).cuda()
st = torch.cuda.current_stream().cuda_stream
s2, s3 = exchange_strides(p, N)
print("strides", s2, s3, p)
g2 = torch.zeros(G * s2, dtype=torch.int64, device="cuda")
g3 = torch.zeros(G * s3, dtype=torch.int64, device="cuda")
c = torch.zeros(6, dtype=torch.int64, device="cuda")
def counters(s):
    s.trace_counters_device(c.data_ptr(), stream=st); torch.cuda.synchronize(); return c.cpu().tolist()
for i, (_, s) in enumerate(ss):
    s.shard_phase1(q.data_ptr(), 32, 128, p, g2.data_ptr() + 8 * i * s2, s2, stream=st)
    print("after p1", i, counters(s))
G2 = g2.cpu().numpy().view(np.uint64)
nz = np.sort(G2[G2 != 0])[::-1]
print("nonzero gathered", nz.size, "thr", hex(nz[p.ndocs - 1]) if nz.size >= p.ndocs else None)
for i, (_, s) in enumerate(ss):
    row = G2[i * s2:(i + 1) * s2]
    print("row", i, "nz", (row != 0).sum(), "ge thr", (row >= nz[p.ndocs - 1]).sum())
for i, (_, s) in enumerate(ss):
    s.shard_phase2(g2.data_ptr(), G, g3.data_ptr() + 8 * i * s3, s3, stream=st)
    print("after p2", i, counters(s))
ids, sc, tr = port.search(whole, qs[0], p)
print("ref", tr)

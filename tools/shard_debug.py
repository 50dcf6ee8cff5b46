"""Debug: per-shard stage-2/3 survivor counts of the global-exact phases vs
the oracle's single-index selections (G=3, N=6000, k=1000)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import oracle  # noqa: E402
import paper_2205_09707_b200 as P  # noqa: E402
from oracle.compare import compose  # noqa: E402
from paper_2205_09707_b200.sharded import exchange_strides, shard_range  # noqa: E402

port = oracle.get("port")
G, N, K = 3, 6000, 512
whole = P.generate_index(N, K, dim=128, nbits=2, mean_len=40, seed=4)
qs = P.generate_queries(whole, 4, seed=21)
ss, bases = [], []
for g in range(G):
    a, b = shard_range(N, G, g)
    hs = P.generate_index(b - a, K, dim=128, nbits=2, mean_len=40, seed=4, pid_base=a)
    ss.append(P.Searcher(P.DeviceIndex.from_host_at(hs, pid_base=a), score_mode=P.ScoreMode.EXACT))
    bases.append((a, b))
p = P.default_params_for_k(1000)
s2, s3 = exchange_strides(p, N)
side = torch.cuda.Stream()
st = side.cuda_stream
for qi, q in enumerate(qs):
    S0, mx0 = port.compute_centroid_scores(whole, q)
    c = compose(port, whole, q, S0, mx0, p)
    k2, k3 = set(map(int, c["k2"])), set(map(int, c["k3"]))
    dq = torch.from_numpy(q.copy()).cuda()
    g2 = torch.zeros(G * s2, dtype=torch.int64, device="cuda")
    g3 = torch.zeros(G * s3, dtype=torch.int64, device="cuda")
    out = torch.zeros(G * (2 * p.k + 2), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    for i, s in enumerate(ss):
        s.shard_phase1(dq.data_ptr(), 32, 128, p, g2.data_ptr() + 8 * i * s2, s2, stream=st)
    for i, s in enumerate(ss):
        s.shard_phase2(g2.data_ptr(), G, g3.data_ptr() + 8 * i * s3, s3, stream=st)
    torch.cuda.synchronize()
    g3h = g3.cpu().numpy().view(np.uint64)
    for i, s in enumerate(ss):
        row = g3h[i * s3:(i + 1) * s3]
        nz = row[row != 0]
        pids = (~(nz & np.uint64(0xFFFFFFFF))).astype(np.uint32) & 0xFFFFFFFF
        a, b = bases[i]
        exp3 = sorted(x for x in k3 if a <= x < b)
        miss = sorted(set(exp3) - set(map(int, pids)))
        print(f"q{qi} shard {i}: exported {nz.size}, global-k3 members {len(exp3)}, missing from export {miss[:5]}")
    # global 1024th key of the union vs counts
    allk = np.sort(g3h[g3h != 0])[::-1]
    t = allk[min(len(allk), 1024) - 1]
    print(f"q{qi}: union {allk.size} keys, keys>=t {int((allk >= t).sum())}")
    for i, s in enumerate(ss):
        s.shard_phase3(g3.data_ptr(), G, out.data_ptr() + 4 * i * (2 * p.k + 2),
                       out.data_ptr() + 4 * (i * (2 * p.k + 2) + p.k), out.data_ptr() + 4 * (i * (2 * p.k + 2) + 2 * p.k),
                       stream=st)
    torch.cuda.synchronize()
    cnt = []
    for s in ss:
        cc = torch.zeros(6, dtype=torch.int64, device="cuda")
        torch.cuda.synchronize()
        s.trace_counters_device(cc.data_ptr())
        torch.cuda.synchronize()
        cnt.append(cc.cpu().tolist())
    print(f"q{qi}: per-shard counters {cnt}; oracle stage2 {len(k2)} stage3 {len(k3)}")

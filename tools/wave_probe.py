"""Throughput-mode (wave engine) probe on a cfg3-shaped synthetic index:
batch timing and, with PLAID_WAVE_TRACE=1, the worker's per-phase times
(median / max over the queries' CTAs, from globaltimer stamps).

    python tools/wave_probe.py [N] [nq] [k] [nbits]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import _native as Nv

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8_800_000
nq = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
k = int(sys.argv[3]) if len(sys.argv) > 3 else 100
nbits = int(sys.argv[4]) if len(sys.argv) > 4 else 1
idx = P.DeviceIndex.synth(N, 1 << 18, dim=128, nbits=nbits, mean_len=68, seed=1)
qs = idx.synth_queries(nq, 32, seed=7)
b = P.BatchSearcher(idx, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(k)
dq = torch.tensor(qs, device="cuda")
pids = torch.zeros(nq * k, dtype=torch.int32, device="cuda")
sc = torch.zeros(nq * k, device="cuda")
n = torch.zeros(nq, dtype=torch.int64, device="cuda")
for it in range(4):
    torch.cuda.synchronize()
    t = time.perf_counter()
    b.search_device(dq.data_ptr(), nq, 32, 128, p, pids.data_ptr(), sc.data_ptr(), n.data_ptr())
    b.sync()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"iter {it}: {dt * 1e3:.1f} ms  {nq / dt:.0f} q/s  wave={b.last_was_wave()} launches={b.last_launches()}",
          flush=True)
c = b.counters(nq)
print("counters mean", c.mean(axis=0), "max", c.max(axis=0))
if os.environ.get("PLAID_WAVE_TRACE"):
    tr = np.zeros((nq, 16), dtype=np.uint64)
    rc = Nv.load().plaid_debug_wave_trace(b._h, tr.ctypes.data_as(C.POINTER(C.c_uint64)), nq)
    assert rc == 0, rc
    spans = [("A probe+kept", 0, 1), ("B-E ranges", 1, 2), ("zero keys", 2, 3), ("sel2", 3, 6),
             ("F stage3", 6, 7), ("sel3", 7, 8), ("G stage4", 8, 9), ("H sort+out", 9, 10)]
    t = tr.astype(np.int64)
    for name, i, j in spans:
        d = (t[:, j] - t[:, i]) / 1e3
        print(f"  {name:14s} median {np.median(d):8.1f} us   max {d.max():8.1f} us")
    for j, name in enumerate(["  range: bounds+prefix", "  range: postings+OR", "  range: compact+count",
                              "  range: scan+score"]):
        d = t[:, 11 + j] / 1e3
        print(f"  {name:22s} median {np.median(d):8.1f} us")
    tot = (t[:, 10] - t[:, 0]) / 1e3
    print(f"  {'CTA total':14s} median {np.median(tot):8.1f} us   max {tot.max():8.1f} us")
    start = t[:, 0] - t[:, 0].min()
    print(f"  CTA starts: median {np.median(start) / 1e3:.1f} us, max {start.max() / 1e3:.1f} us")

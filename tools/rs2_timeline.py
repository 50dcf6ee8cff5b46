"""Phase timeline of the latency path's range_stage2 kernel (one CTA per pid
range) on a cfg2-shaped synthetic index: median / max over the CTAs of each
phase, from globaltimer stamps (plaid_debug_rs2_trace).

    python tools/rs2_timeline.py [N] [k]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import _native as Nv

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8_800_000
k = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
idx = P.DeviceIndex.synth(N, 1 << 18, dim=128, nbits=2, mean_len=68, seed=1)
qs = idx.synth_queries(8, 32, seed=7)
s = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(k)
lib = Nv.load()
for q in qs[:4]:
    s.search(q, p)  # warm-up
lib.plaid_debug_rs2_trace(1, None)
R = (N + 65535) // 65536
rows = []
for q in qs[4:]:
    s.search(q, p)
    out = np.zeros(512 * 8, dtype=np.uint64)
    assert lib.plaid_debug_rs2_trace(0, out.ctypes.data_as(C.c_void_p)) == 0
    rows.append(out.reshape(512, 8)[:R].astype(np.int64))
lib.plaid_debug_rs2_trace(0, None)
t = np.concatenate(rows)
names = [("PDL wait", 6, 0), ("runs located", 0, 1), ("postings", 1, 2), ("compaction", 2, 3),
         ("kept masks", 3, 4), ("zero keys + list", 4, 7), ("scoring", 7, 5)]
for name, a, b in names:
    d = (t[:, b] - t[:, a]) / 1e3
    print(f"{name:26s} median {np.median(d):7.2f} us   max {d.max():7.2f} us")
start = t[:, 0] - t[:, 0].min(axis=0)
for qi, r in enumerate(rows):
    span = (r[:, 5].max() - r[:, 0].min()) / 1e3
    print(f"query {qi}: CTA span {span:.1f} us (first start to last end)")
r = s.search(qs[0], p)
tr = r.trace.counters()
print("trace:", tr)
print(f"kept-token hits per C1 member: {tr['stage2_rows_gathered'] / max(tr['stage1_candidates'], 1):.2f}, "
      f"per range: {tr['stage2_rows_gathered'] / R:.0f}")

"""Tensor-core stage-4 timeline (per-CTA globaltimer stamps, rank128.cu
s4_stamp): one cfg2 query, L2 flushed, printed as medians / maxima of each
phase relative to the kernel's first CTA start.  Run under gpurun."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200 import _native  # noqa: E402

cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"])
h = bench.make_index(cfg, 0)
idx = P.DeviceIndex.from_host(h)
s = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
p = bench.params_for(cfg)
qs = P.generate_queries(h, 8, seed=1234)
lib = _native.load()
lib.plaid_debug_s4_set.argtypes = [C.c_uint32]
lib.plaid_debug_s4_trace.argtypes = [C.c_void_p]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
names = ["start", "prefetched", "B landed", "t0 A stored", "t0 D ready", "t0 epi done", "t1 A stored", "t1 D ready",
         "t1 epi done", "t2 A stored", "t2 D ready", "t2 epi done", "end"]
for it in range(6):
    flush.zero_()
    torch.cuda.synchronize()
    lib.plaid_debug_s4_set(1 if it == 5 else 0)
    r = s.search(qs[it], p)
tr = np.zeros(512 * 16, dtype=np.uint64)
lib.plaid_debug_s4_trace(tr.ctypes.data)
tr = tr.reshape(512, 16).astype(np.int64)
live = tr[:, 0] > 0
t0 = tr[live, 0].min()
print(f"CTAs with stamps: {live.sum()}, T4 = {r.trace.decompressed_tokens}")
for e, nm in enumerate(names):
    v = tr[live, e]
    v = v[v > 0] - t0
    if v.size:
        print(f"{nm:14s} n={v.size:4d} median {np.median(v) / 1e3:7.2f} us  max {v.max() / 1e3:7.2f} us")

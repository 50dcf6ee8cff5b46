"""Stage-4 (stream_fused) timeline of CTA 0: run with PLAID_RANK_DBG=1 on a GPU."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200 import _native  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
h = P.generate_index(N, 1 << 18, dim=128, nbits=2, mean_len=68, seed=0)
qs = P.generate_queries(h, 4)
idx = P.DeviceIndex.from_host(h)
s = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(1000)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for i in range(6):
    flush.zero_()
    torch.cuda.synchronize()
    s.search(qs[i % 4], p)
    ms.append(round(s.phase_ms()["stage4_rank"], 4))
print("stage4_ms", ms)
L = _native.load()
buf = (ctypes.c_ulonglong * 320)()
L.plaid_debug_rank_trace(buf)
a = np.array(buf, dtype=np.int64).reshape(5, 64)
t0 = a[0, 0]
for k in range(8):
    if a[0, k] == 0:
        break
    print(k, " ".join(f"{n}={(a[i, k] - t0) / 1000:6.2f}" for i, n in enumerate(["p_start", "p_rows", "p_done", "c_start", "c_done"])))

"""Stage-1 tensor kernel timeline (debug): run with PLAID_TF32_DBG=16 on a GPU.

Prints per-chunk pipeline stamps of CTA 0 (TMA issue, raw tile landed, lo
buffer free, split done, MMA start), per-tile accumulator-full / epilogue-done
times, and the spread of per-CTA begin/end times.
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200 import _native  # noqa: E402

h = P.generate_index(200000, 1 << 18, dim=128, nbits=2, mean_len=8, seed=0)
qs = P.generate_queries(h, 4)
idx = P.DeviceIndex.from_host(h)
s = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR)
p = P.default_params_for_k(1000)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ms = []
for i in range(8):
    flush.zero_()
    torch.cuda.synchronize()
    s.search(qs[i % 4], p)
    ms.append(s.phase_ms()["scores"])
print("scores_ms", ms)
L = _native.load()
buf = (ctypes.c_ulonglong * 2560)()
L.plaid_debug_tf32_trace(buf)
a = np.array(buf, dtype=np.int64)
ev = a[:2048].reshape(8, 256)
cta = a[2048:].reshape(2, 256)
t0 = ev[0, 0]
names = ["issue", "rawfull", "opsfree", "conv_done", "mmastart"]
for g in list(range(0, 8)) + list(range(48, 56)):
    print(g, " ".join(f"{n}={(ev[i, g] - t0) / 1000:7.2f}" for i, n in enumerate(names)),
          f"conv3_done={(ev[7, g] - t0) / 1000:7.2f}")
for lt in range(16):
    print("tile", lt, f"tfull={(ev[5, lt] - t0) / 1000:7.2f} epidone={(ev[6, lt] - t0) / 1000:7.2f}")
nz = cta[0] > 0
b, e = cta[0][nz], cta[1][nz]
print(f"ctas={nz.sum()} begin spread={(b.max() - b.min()) / 1000:.2f}us "
      f"end spread={(e.max() - e.min()) / 1000:.2f}us span={(e.max() - b.min()) / 1000:.2f}us")

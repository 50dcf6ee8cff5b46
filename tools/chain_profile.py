"""Marginal cost of each kernel inside the PDL-chained search (cfg2 by
default): the same device-timed step as bench.py (L2 flushed before every
query, CUDA events on the search stream), with the search truncated after its
first `cap` launches (plaid_debug_set_launch_cap), cap = 1 .. full.  The
difference between consecutive caps is what that kernel adds to the real
chain — unlike ncu's serialised launch list, overlap with its neighbours
(PDL prologues, tails) is included.  Results of truncated searches are
garbage; only the times are read.  Run under gpurun:

    python tools/chain_profile.py [cfg2] [steps] [caps, e.g. 0,1,2]
"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_2205_09707_b200 as P  # noqa: E402
from paper_2205_09707_b200 import _native  # noqa: E402

import os

PAD = int(os.environ.get("PAD_CYCLES", "0"))
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cfg = dict(bench.CONFIGS[name])
h = bench.make_index(cfg, 0)
idx = P.DeviceIndex.from_host(h)
p = bench.params_for(cfg)
qs = P.generate_queries(h, 64, seed=1234)
lib = _native.load()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
sh = stream.cuda_stream
dq = [torch.from_numpy(q).cuda() for q in qs]
d_pids = torch.zeros(p.k, dtype=torch.int32, device="cuda")
d_scores = torch.zeros(p.k, dtype=torch.float32, device="cuda")
d_n = torch.zeros(1, dtype=torch.int64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

s = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR, record_times=False, use_graphs=False)
s.search_device(dq[0].data_ptr(), 1, 32, 128, p, d_pids.data_ptr(), d_scores.data_ptr(), d_n.data_ptr(), stream=sh)
torch.cuda.synchronize()
full = s.last_launches()


def timed(cap):
    lib.plaid_debug_set_launch_cap(cap)
    # a fresh searcher per cap: kernels that never run leave no stale state
    # behind for the ones that do
    t = P.Searcher(idx, score_mode=P.ScoreMode.TENSOR, record_times=False, use_graphs=False)
    ms, host = [], []
    for i in range(steps + 5):
        flush.zero_()
        if PAD:  # keep the GPU busy until the whole chain is enqueued (host-bound check)
            torch.cuda._sleep(PAD)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        h0 = time.perf_counter()
        t.search_device(dq[i % 64].data_ptr(), 1, 32, 128, p, d_pids.data_ptr(), d_scores.data_ptr(),
                        d_n.data_ptr(), stream=sh)
        h1 = time.perf_counter()
        b.record(stream)
        b.synchronize()
        if i >= 5:
            ms.append(a.elapsed_time(b) * 1e3)
            host.append((h1 - h0) * 1e6)
    lib.plaid_debug_set_launch_cap(-1)
    t.close()
    return float(np.median(ms)), float(np.min(ms)), float(np.median(host))


print(f"{name}: {full} launches per search; median / min step us with the chain cut after each launch")
prev = 0.0
caps = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else list(range(0, full + 1))
for cap in caps:
    med, mn, hst = timed(cap)
    print(f"cap {cap:2d}: median {med:7.2f} us  min {mn:7.2f}  marginal {med - prev:+7.2f}  (host enqueue {hst:6.1f} us)")
    prev = med

"""Where the host API's end-to-end time goes (GPU box): the full
Searcher.search call, the bare C-ABI call with preallocated buffers, and the
device-timed step, on a small index (cfg1 scale) and cfg2 params."""
import ctypes as C
import statistics
import time

import numpy as np
import torch

import paper_2205_09707_b200 as P
from paper_2205_09707_b200 import _native as N

h = P.generate_index(10000, 4096, dim=128, nbits=2, mean_len=64, seed=1)
qs = P.generate_queries(h, 8, seed=2)
idx = P.DeviceIndex.from_host(h, device=0)
s = P.Searcher(idx, device=0, score_mode=P.ScoreMode.TENSOR, record_times=False)
p = P.default_params_for_k(10)
lib = N.load()


def med(f, n=300):
    for _ in range(20):
        f()
    ts = []
    for i in range(n):
        t0 = time.perf_counter()
        f()
        ts.append(time.perf_counter() - t0)
    return 1e6 * statistics.median(ts)


q = np.ascontiguousarray(qs[0])
ids = np.empty(p.k, dtype=np.uint32)
sc = np.empty(p.k, dtype=np.float32)
n = C.c_uint64()
tr = N.Trace()
cp = p._c(False)
qa, ia, sa = (x.__array_interface__["data"][0] for x in (q, ids, sc))
print(f"Searcher.search      {med(lambda: s.search(q, p)):7.1f} us")
print(f"bare plaid_search    {med(lambda: lib.plaid_search(s._h, qa, q.shape[0], q.shape[1], C.byref(cp), ia, sa, C.byref(n), C.byref(tr))):7.1f} us")
print(f"  (no trace)         {med(lambda: lib.plaid_search(s._h, qa, q.shape[0], q.shape[1], C.byref(cp), ia, sa, C.byref(n), None)):7.1f} us")
dq = torch.from_numpy(q).cuda()
dp = torch.empty(p.k, dtype=torch.int32, device="cuda")
ds = torch.empty(p.k, dtype=torch.float32, device="cuda")
dn = torch.empty(1, dtype=torch.int64, device="cuda")
st = torch.cuda.Stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
def dev():
    with torch.cuda.stream(st):
        a.record(st)
        s.search_device(dq.data_ptr(), 1, q.shape[0], q.shape[1], p, dp.data_ptr(), ds.data_ptr(), dn.data_ptr(), st.cuda_stream)
        b.record(st)
    b.synchronize()
    return a.elapsed_time(b)
for _ in range(20):
    dev()
print(f"device step          {1e3 * statistics.median([dev() for _ in range(300)]):7.1f} us")
print(f"search_device+sync   {med(lambda: (s.search_device(dq.data_ptr(), 1, q.shape[0], q.shape[1], p, dp.data_ptr(), ds.data_ptr(), dn.data_ptr(), st.cuda_stream), st.synchronize())):7.1f} us")

import torch
x = torch.randn(1 << 25, device="cuda")  # 128 MiB fp32 (= C at K=2^18)
y = torch.empty_like(x)
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, n=10):
    ms = []
    for _ in range(n):
        fl.zero_(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(); fn(); b.record(); b.synchronize(); ms.append(a.elapsed_time(b))
    return sorted(ms)[n // 2]
for name, fn, by in [("sum", lambda: x.sum(), 1), ("copy", lambda: y.copy_(x), 2), ("amax", lambda: x.amax(), 1)]:
    m = t(fn)
    print(f"{name}: {m*1e3:.1f} us  {by * x.numel() * 4 / m / 1e6:.0f} GB/s")

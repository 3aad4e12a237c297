import torch, time
n = 2563201
h1 = torch.randn(n, dtype=torch.complex128).pin_memory(); h2 = torch.randn(n, dtype=torch.complex128).pin_memory()
d1 = torch.empty(n, dtype=torch.complex128, device="cuda"); d2 = torch.empty_like(d1)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, k=20):
    fn(); torch.cuda.synchronize(); t0=time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter()-t0)/k*1e3
nb = n*16
ms = t(lambda: d1.copy_(h1, non_blocking=True)); print("H2D 41MB", ms, nb/ms/1e6, "GB/s")
ms = t(lambda: h1.copy_(d1, non_blocking=True)); print("D2H 41MB", ms, nb/ms/1e6, "GB/s")
def two():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2, non_blocking=True)
ms = t(two); print("2x H2D concurrent", ms, 2*nb/ms/1e6, "GB/s")
def seq():
    d1.copy_(h1, non_blocking=True); d2.copy_(h2, non_blocking=True); h1.copy_(d1, non_blocking=True)
ms = t(seq); print("H2D+H2D+D2H serial", ms, 3*nb/ms/1e6, "GB/s")

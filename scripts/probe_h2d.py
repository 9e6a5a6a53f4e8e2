"""H2D of one C3 scan (131072 f64 ranges + uint8 validity, 1.18 MB): pageable
copies vs a memcpy into pinned staging + DMA (medians of 200, us)."""
import time, numpy as np, torch, statistics
n = 131072
r = np.random.rand(n)
v = (np.random.rand(n) < 0.5)
g = torch.empty(n, dtype=torch.float64, device="cuda")
gv = torch.empty(n, dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
pinv = torch.empty(n, dtype=torch.uint8, pin_memory=True)
pn = pin.numpy(); pvn = pinv.numpy()
def t(fn, k=200):
    for _ in range(20): fn()
    ts=[]
    for _ in range(k):
        a=time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append((time.perf_counter()-a)*1e6)
    return round(statistics.median(ts),1)
print("pageable", t(lambda: (g.copy_(torch.from_numpy(r), non_blocking=True), gv.copy_(torch.from_numpy(v.view(np.uint8)), non_blocking=True))))
def pinned():
    np.copyto(pn, r); np.copyto(pvn, v.view(np.uint8))
    g.copy_(pin, non_blocking=True); gv.copy_(pinv, non_blocking=True)
print("pinned staging", t(pinned))
print("memcpy only", t(lambda: (np.copyto(pn, r), np.copyto(pvn, v.view(np.uint8)))))
print("pinned dma only", t(lambda: (g.copy_(pin, non_blocking=True), gv.copy_(pinv, non_blocking=True))))

"""Host<->device copy rates for one 7 MB vector on the box: pageable vs pinned."""
import time, torch, numpy as np
n = 884736
d = torch.empty(n, dtype=torch.float64, device="cuda")
pg = torch.rand(n, dtype=torch.float64)
pn = torch.rand(n, dtype=torch.float64).pin_memory()
for name, src in (("pageable", pg), ("pinned", pn)):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(10):
            d.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        print(name, "h2d", (time.perf_counter() - t) / 10 * 1e3, "ms")
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(10):
            src.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        print(name, "d2h", (time.perf_counter() - t) / 10 * 1e3, "ms")
big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
dbig = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); dbig.copy_(big, non_blocking=True); torch.cuda.synchronize()
print("pinned 256MB h2d GB/s", 256 * 1.048576e6 / (time.perf_counter() - t) / 1e9)

"""Does a small device->host read wait for a large host->device copy in
flight? pageable vs pinned destination (decides how the library reads sizes)."""
import time

import torch

n = 3 << 30  # 24 GB of int64? use 3 Gi elements of int64 = 24 GB
h = torch.empty(n, dtype=torch.int64, pin_memory=True)
d = torch.empty(n, dtype=torch.int64, device="cuda")
small = torch.arange(4, dtype=torch.int64, device="cuda")
pinned = torch.empty(4, dtype=torch.int64, pin_memory=True)
side = torch.cuda.Stream()
other = torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
full = time.perf_counter() - t0
print(f"H2D {n * 8 / 1e9:.1f} GB alone: {full * 1e3:.1f} ms = {n * 8 / full / 1e9:.1f} GB/s")
for mode in ("pageable", "pinned"):
    torch.cuda.synchronize()
    with torch.cuda.stream(side):
        d.copy_(h, non_blocking=True)
    time.sleep(0.01)
    t1 = time.perf_counter()
    with torch.cuda.stream(other):
        if mode == "pageable":
            x = small.cpu()
        else:
            pinned.copy_(small, non_blocking=True)
            other.synchronize()
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{mode:9s} small D2H during the H2D: {(t2 - t1) * 1e3:.2f} ms (copy finished {(t3 - t1) * 1e3:.1f} ms after)")

"""Time the host<->device pieces of the e2e plugin call on this box."""
import time

import torch

s = torch.cuda.Stream()
for nbytes in (409600, 393216, 4096, 8192, 16384):
    h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    for direction in ("h2d", "d2h"):
        for _ in range(10):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        for _ in range(100):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e1.record()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        print(f"{direction} {nbytes} B: {e0.elapsed_time(e1) / 100 * 1e3:.2f} us device, "
              f"{(t1 - t0) / 100 * 1e6:.2f} us wall")
# sync round trip
e = torch.cuda.Event()
t0 = time.perf_counter()
for _ in range(100):
    torch.cuda._sleep(1)
    torch.cuda.synchronize()
print(f"launch+sync round trip {(time.perf_counter() - t0) / 100 * 1e6:.2f} us")

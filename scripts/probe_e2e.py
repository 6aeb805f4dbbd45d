"""Where the e2e plugin call's time over the device round goes: wall time per
graph launch + synchronise of (a) one empty kernel, (b) the round's four H2D
copies (409,600 B from pinned memory), (c) (b) plus a device kernel reading
the same bytes from mapped pinned memory instead, (d) mapped-memory read only."""
import time

import torch

torch.cuda.init()
s = torch.cuda.Stream()
sizes = (393216, 4096, 4096, 8192)
hs = [torch.empty(n, dtype=torch.uint8).pin_memory() for n in sizes]
ds = [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes]
tiny = torch.zeros(1, device="cuda")


def timed(fn, reps=200):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            fn()
    for _ in range(20):
        g.replay()
        torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        g.replay()
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def empty():
    tiny.add_(1)


def copies():
    for h, d in zip(hs, ds):
        d.copy_(h, non_blocking=True)
    tiny.add_(1)


def one_copy():
    ds[0].copy_(hs[0], non_blocking=True)
    tiny.add_(1)


print(f"empty kernel graph + sync: {timed(empty):.1f} us")
print(f"4 H2D copies graph + sync: {timed(copies):.1f} us")
print(f"1 H2D copy (393 KB) graph + sync: {timed(one_copy):.1f} us")

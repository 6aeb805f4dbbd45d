"""Time k_refresh on the c3 storm for an experiment build (--lib)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
a = ap.parse_args()
_lib.load(a.lib)
n, nbins, k = 200_000, 512, 64
g = torch.Generator(device="cuda")
g.manual_seed(0)
d = "cuda"
lens = torch.clamp(torch.round(torch.exp(5.5 + 0.8 * torch.randn((n, k), generator=g, device=d))), 1, 2048).to(torch.int32)
I = torch.randint(1, 4097, (n,), generator=g, device=d, dtype=torch.int32)
gg = torch.where(torch.rand(n, generator=g, device=d) < 0.4, torch.randint(0, 2049, (n,), generator=g, device=d), 0).to(torch.int32)
comp = torch.ones((n, k), dtype=torch.int64, device=d)
fb = torch.zeros((3, nbins), dtype=torch.int64, device=d)
npts = torch.zeros(n, dtype=torch.int32, device=d)
pbin = torch.zeros((n, nbins), dtype=torch.int32, device=d)
pcnt = torch.zeros((n, nbins), dtype=torch.int32, device=d)
pD = torch.zeros((n, nbins), dtype=torch.int64, device=d)
G = torch.zeros(n, dtype=torch.float64, device=d)
P = lambda t: t.data_ptr()  # noqa: E731
_lib.call("ss_finish", P(comp), P(lens), n, k, 1, 2048, nbins, P(I), P(fb[0]), P(fb[1]), P(fb[2]), nbins,
          P(npts), P(pbin), P(pcnt), P(pD), None, None, P(G), _lib.stream_ptr())
bucket = torch.zeros(n, dtype=torch.int32, device=d)
G0 = None
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(50):
        _lib.call("ss_refresh", n, P(I), P(gg), P(bucket), 200, P(npts), P(pcnt), P(pD), nbins, P(G), None, 1, _lib.stream_ptr())
    e1.record()
    torch.cuda.synchronize()
print(f"{a.lib}: k_refresh {e0.elapsed_time(e1) / 50 * 1e3:.1f} us  G checksum {G.sum().item():.6e}")

"""Time ss_rank at several n for one library build (CUDA events, graph-free)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
a = ap.parse_args()
_lib.load(a.lib)
from paper_2603_07917_b200.scheduler import rank  # noqa: E402

out = []
for n in (1024, 2048, 3000, 4096, 6000, 8192):
    rng = np.random.default_rng(n)
    G = torch.as_tensor(rng.uniform(1, 1e7, n), device="cuda")
    ids = torch.arange(n, device="cuda", dtype=torch.int64)
    perm = torch.empty(n, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(_lib.lib().ss_rank_workspace_bytes(n)), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            rank(G, ids, perm, ws)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(50):
            rank(G, ids, perm, ws)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    out.append(f"n={n}: {e0.elapsed_time(e1) / 200 * 1e3:.1f}")
print(a.lib, "  ".join(out))

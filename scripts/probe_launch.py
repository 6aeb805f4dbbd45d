"""Launch + synchronise overhead per piece of the c2 round: wall time of
(graph replay + synchronize) vs the GPU time between events around it, for
a graph of (a) the similarity kernel alone, (b) the whole device round,
(c) a trivial kernel."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler  # noqa: E402
from paper_2603_07917_b200.synthetic import make_bank_device, make_queries  # noqa: E402

_lib.load()
n_bank, nq = 1 << 20, 1024
emb, lens, _ = make_bank_device(n_bank, 384, 4096, 0)
win = HistoryWindow(n_bank, 384)
win.push(emb, lens)
q, qi, I, ids = make_queries(nq, 384, 4096, 0, qseed=1000)
dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
sched = SageScheduler(win, RoundConfig(k=64, theta=0.8, min_matches=20, max_len=2048, nbins=128))
part = torch.empty(64 * nq * 64, dtype=torch.int64, device="cuda")
ns = ctypes.c_int32()
lib = _lib.lib()
tiny = torch.zeros(1, device="cuda")


def topk():
    lib.ss_topk_partials(win.handle, dq.data_ptr(), dqi.data_ptr(), nq, 64, ctypes.c_float(0.8),
                         _lib.ALGO["tcgen05"], part.data_ptr(), 64, ctypes.byref(ns), _lib.stream_ptr())


def graph_of(fn):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    return g


def measure(name, g, reps=400):
    for _ in range(20):
        g.replay()
        torch.cuda.synchronize()
    wall = np.empty(reps)
    gpu = np.empty(reps)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(reps):
        t0 = time.perf_counter()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        wall[i] = (time.perf_counter() - t0) * 1e6
        gpu[i] = e0.elapsed_time(e1) * 1e3
    print(f"{name:28s} wall median {np.median(wall):7.1f} p10 {np.percentile(wall, 10):7.1f}   "
          f"gpu median {np.median(gpu):7.1f} p10 {np.percentile(gpu, 10):7.1f}   "
          f"overhead median {np.median(wall - gpu):6.1f}")


measure("trivial kernel", graph_of(lambda: tiny.add_(1)))
measure("similarity kernel alone", graph_of(topk))
g_round, _ = sched.capture_round(dq, dqi, dI, dids)
measure("device round", g_round)
measure("similarity kernel alone", graph_of(topk))
measure("device round", g_round)

"""Per-call wall time of the host-buffer plugin call (ss_schedule_round_host)
on the c2 round for one library build: median / mean / p10 of N calls.

    python scripts/time_e2e.py --lib build_exp/NAME/libsagesched.so [--calls 2000]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lib", default=None)
ap.add_argument("--calls", type=int, default=2000)
a = ap.parse_args()
_lib.load(a.lib)
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler  # noqa: E402
from paper_2603_07917_b200.synthetic import make_bank_device, make_queries  # noqa: E402

n_bank, nq = 1 << 20, 1024
emb, lens, _ = make_bank_device(n_bank, 384, 4096, 0)
win = HistoryWindow(n_bank, 384)
win.push(emb, lens)
q, qi, I, ids = make_queries(nq, 384, 4096, 0, qseed=1000)
sched = SageScheduler(win, RoundConfig(k=64, theta=0.8, min_matches=20, max_len=2048, nbins=128))


def pin(x):
    return torch.from_numpy(np.ascontiguousarray(x)).pin_memory().numpy()


hq, hqi, hI, hids = pin(q), pin(qi), pin(I), pin(ids)
G = torch.empty(nq, dtype=torch.float64).pin_memory().numpy()
perm = torch.empty(nq, dtype=torch.int64).pin_memory().numpy()
s = torch.cuda.Stream()
for _ in range(20):
    sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s)
ts = np.empty(a.calls)
for i in range(a.calls):
    t0 = time.perf_counter()
    sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s)
    ts[i] = time.perf_counter() - t0
ts *= 1e6
dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
graph, _ = sched.capture_round(dq, dqi, dI, dids)
td = np.empty(a.calls // 2)
for i in range(len(td)):
    t0 = time.perf_counter()
    graph.replay()
    torch.cuda.synchronize()
    td[i] = time.perf_counter() - t0
td *= 1e6
print(f"device-resident graph replay + sync: median {np.median(td):.1f} us")
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
for e0, e1 in ev:
    e0.record()
    graph.replay()
    e1.record()
    torch.cuda.synchronize()
gd = np.array([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev])
print(f"  same, GPU-side (events around each replay): median {np.median(gd):.1f} us")
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    graph.replay()
e1.record()
torch.cuda.synchronize()
tl = np.empty(200)
for i in range(200):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    graph.replay()
    tl[i] = time.perf_counter() - t0
torch.cuda.synchronize()
ev1 = torch.cuda.Event()
tq = np.empty(500)
for i in range(500):
    t0 = time.perf_counter()
    graph.replay()
    ev1.record()
    while not ev1.query():
        pass
    tq[i] = time.perf_counter() - t0
print(f"  replay + spin on event.query(): median {np.median(tq) * 1e6:.1f} us")
print(f"  host time inside graph.replay(): median {np.median(tl) * 1e6:.1f} us")
import ctypes  # noqa: E402
cudart = ctypes.CDLL("libcudart.so.12") if False else None
print(f"  back-to-back replays: {e0.elapsed_time(e1) * 1e3 / 200:.1f} us per round")
print(f"{a.lib}: median {np.median(ts):.1f} us  mean {ts.mean():.1f}  p10 {np.percentile(ts, 10):.1f}  "
      f"p90 {np.percentile(ts, 90):.1f}  G sum {G.sum():.6e}  perm[0] {perm[0]}")

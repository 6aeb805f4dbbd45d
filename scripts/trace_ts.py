"""Per-tile timeline of CTA (0,0) of k_topk_ts from an SS_TRACE build."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.synthetic import make_bank_device, make_queries  # noqa: E402

lib_path, nq, theta = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
_lib.load(lib_path)
raw = C.CDLL(lib_path)
rows = 1 << 20
emb, lens, _ = make_bank_device(rows, 384, 4096, 0)
w = HistoryWindow(rows, 384)
w.push(emb, lens)
q, qi, _, _ = make_queries(nq, 384, 4096, 0, 1000)
dq, dqi = torch.as_tensor(q, device="cuda"), torch.as_tensor(qi, device="cuda")
part = torch.empty(1024 * nq * 64, dtype=torch.int64, device="cuda")
ns = C.c_int32()
for i in range(3):
    if i == 2:
        torch.cuda.synchronize()
        raw.ss_exp_trace_reset()
    _lib.call("ss_topk_partials", w.handle, dq.data_ptr(), dqi.data_ptr(), nq, 64, float(np.float32(theta)),
              _lib.ALGO["tcgen05"], part.data_ptr(), 1024, C.byref(ns), _lib.stream_ptr())
torch.cuda.synchronize()
tr = np.zeros((9, 512), dtype=np.int64)
wt = np.zeros((5, 12, 512), dtype=np.int64)
assert raw.ss_exp_trace(tr.ctypes.data_as(C.c_void_p), wt.ctypes.data_as(C.c_void_p)) == 0
T = 300 if nq == 1024 else 200
t0 = tr[5][0]
tr = tr - t0
wt = wt - t0
a, b = 20, T - 20
per = np.diff(tr[5][a:b + 1])
print(f"tile period (MMA wait start to next) mean {per.mean():.0f} cycles, p10 {np.percentile(per,10):.0f} p90 {np.percentile(per,90):.0f}")
def m(x):
    return f"{np.mean(x):7.0f} (p90 {np.percentile(x, 90):6.0f})"
print("MMA: wait full", m(tr[6][a:b] - tr[5][a:b]), " issue 12 MMAs + commits", m(tr[7][a:b] - tr[6][a:b]))
print("EPI: pre (bounds)", m(tr[1][a:b] - tr[4][a - 1:b - 1]) + " [vs last warp]", " wait tfull", m(tr[2][a:b] - tr[1][a:b]),
      " pull+release", m(tr[3][a:b] - tr[2][a:b]), " filter", m(tr[4][a:b] - tr[3][a:b]))
print("tfull seen by epi after MMA issue end:", m(tr[2][a:b] - tr[7][a:b]))
print("release(t) -> MMA full wait end (t+2):", m(tr[6][a + 2:b + 2] - tr[3][a:b]))
print("producer part0 issue (t) -> MMA wait end (t):", m(tr[6][a:b] - tr[8][a:b]))
print("producer part0 issue (t) vs MMA(t-2) issue end:", m(tr[8][a:b] - tr[7][a - 2:b - 2]))
rel = wt[2][:, a:b] - wt[2][:, a:b].min(axis=0)  # release lag behind the first warp
def row(name, x):
    print(f"{name:34s}", " ".join(f"{int(v):5d}" for v in np.round(x.mean(axis=1))))
print(f"{'per epilogue warp (2..13)':34s}", " ".join(f"{w:5d}" for w in range(2, 14)))
row("release lag behind first warp", rel)
print(f"{'releases last (count)':34s}", " ".join(f"{v:5d}" for v in np.bincount(np.argmax(wt[2][:, a:b], axis=0), minlength=12)))
row("ifull wait (prev filter end -> 0)", wt[4][:, a:b] - wt[3][:, a - 1:b - 1])
row("bounds (0 -> 1)", wt[0][:, a:b] - wt[4][:, a:b])
row("tfull wait (1 -> 2)", wt[1][:, a:b] - wt[0][:, a:b])
row("pull + release (2 -> 3)", wt[2][:, a:b] - wt[1][:, a:b])
row("filter (3 -> 4)", wt[3][:, a:b] - wt[2][:, a:b])
for t in range(100, 104):
    print(t, {k: int(tr[k][t]) for k in range(1, 9)})

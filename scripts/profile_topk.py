"""Set up the bench workload and launch the similarity kernel alone, for ncu.

    python scripts/profile_topk.py --nq 1024 --algo tcgen05 --reps 3
"""

import argparse
import ctypes as C
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.synthetic import inv_norm_np, make_bank_device, make_queries  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 20)
    ap.add_argument("--nq", type=int, default=1024)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--theta", type=float, default=0.8)
    ap.add_argument("--algo", default="tcgen05")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--time", action="store_true")
    ap.add_argument("--lib", default=None, help="an experiment build of libsagesched.so")
    ap.add_argument("--random", action="store_true",
                    help="uniform random int8 queries (few neighbours above 0.8: the pure top-k "
                         "cascade's worst case)")
    a = ap.parse_args()
    _lib.load(a.lib)
    emb, lens, _ = make_bank_device(a.rows, 384, 4096, 0)
    w = HistoryWindow(a.rows, 384)
    w.push(emb, lens)
    del emb
    q, qi, _, _ = make_queries(a.nq, 384, 4096, 0, 1000)
    if a.random:
        q = np.random.default_rng(7).integers(-60, 61, (a.nq, 384)).astype(np.int8)
        qi = inv_norm_np(q)
    dq, dqi = torch.as_tensor(q, device="cuda"), torch.as_tensor(qi, device="cuda")
    part = torch.empty(1024 * a.nq * a.k, dtype=torch.int64, device="cuda")
    ns = C.c_int32()

    def launch():
        _lib.call("ss_topk_partials", w.handle, dq.data_ptr(), dqi.data_ptr(), a.nq, a.k,
                  float(np.float32(a.theta)), _lib.ALGO[a.algo], part.data_ptr(), 1024,
                  C.byref(ns), _lib.stream_ptr())

    launch()
    torch.cuda.synchronize()
    if a.time:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        ops = 2.0 * a.nq * a.rows * 384
        print(f"nq={a.nq} rows={a.rows} algo={a.algo} slices={ns.value}: {ms:.4f} ms "
              f"{ops / ms / 1e9:.1f} TOPS  bank {a.rows * 388 / ms / 1e6:.1f} GB/s")
    else:
        for _ in range(a.reps):
            launch()
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()

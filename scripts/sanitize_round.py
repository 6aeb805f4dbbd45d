"""One small scheduling round of every stage-1 kernel instantiation plus the
merge/finish/rank kernels, for compute-sanitizer (racecheck / memcheck /
synccheck).  Kept small: the sanitizers replay every access.

    compute-sanitizer --tool racecheck python scripts/sanitize_round.py
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import sagesched_oracle as O  # noqa: E402
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler  # noqa: E402


def main():
    _lib.load()
    n = 6000
    emb, lens, _, _ = O.make_bank(n + 300, 384, 30, 3)
    w = HistoryWindow(n, 384)
    w.push(emb[:n], lens[:n])
    I = np.random.default_rng(1).integers(1, 4097, 300).astype(np.int32)
    ok = True
    # nq = 300: k_topk_ts (theta 0.8: locked shared heaps; theta -1: the
    # pure top-k cascade -- threshold pass, then the SHARE instantiation for
    # unresolved tiles, forced by random queries) + k_merge_finish_w + rank;
    # nq = 64: k_topk_tc
    rq = np.random.default_rng(2).integers(-60, 61, (300, 384)).astype(np.int8)
    for nq, theta, rand in ((300, 0.8, False), (300, -1.0, False), (300, -1.0, True), (64, 0.8, False),
                            (64, -1.0, False)):
        q = rq[:nq] if rand else emb[n:n + nq]
        qi = O.inv_norm(q)
        cfg = RoundConfig(k=32, theta=theta, min_matches=20, nbins=64)
        perm, G, _ = SageScheduler(w, cfg).schedule_round(
            torch.as_tensor(q, device="cuda"), torch.as_tensor(qi, device="cuda"),
            torch.as_tensor(I[:nq], device="cuda"), torch.arange(nq, device="cuda"))
        torch.cuda.synchronize()
        keys = O.scores(q, qi, emb[:n], O.inv_norm(emb[:n]))
        ref = O.predict_round(keys, np.arange(n), lens[:n], I[:nq], 32, theta, 20, 2048, 64,
                              window_lens=lens[:n])
        good = np.array_equal(G.cpu().numpy(), np.array([r["G"] for r in ref]))
        print(f"nq={nq} theta={theta}{' random queries' if rand else ''}: {'ok' if good else 'MISMATCH'}")
        ok &= good
    # the slice merge (k_merge_w) behind HistoryWindow.topk, and the shard
    # merge of two half-bank windows (ss_merge_topk) against the full bank
    from paper_2603_07917_b200.sharded import ShardPlan
    q = torch.as_tensor(emb[n:n + 300], device="cuda")
    qi = torch.as_tensor(O.inv_norm(emb[n:n + 300]), device="cuda")
    c0, l0 = w.topk(q, qi, 32, 0.6)
    comps, lns = [], []
    for r in range(2):
        plan = ShardPlan(n, 2, r)
        ws = HistoryWindow(plan.local_capacity, 384, global_capacity=n, slot_offset=plan.slot_offset)
        idx, seq, slot = plan.route(0, n)
        ws.write(torch.as_tensor(emb[idx], device="cuda"), torch.as_tensor(lens[idx], device="cuda"),
                 torch.as_tensor(seq, device="cuda"), torch.as_tensor(slot, device="cuda"))
        ws.set_head(n)
        c, l_ = ws.topk(q, qi, 32, 0.6)
        comps.append(c)
        lns.append(l_)
    cx, lx = torch.stack(comps).contiguous(), torch.stack(lns).contiguous()
    mc, ml = torch.empty_like(c0), torch.empty_like(l0)
    _lib.call("ss_merge_topk", _lib.ptr(cx), _lib.ptr(lx), 2, 300, 32, _lib.ptr(mc), _lib.ptr(ml),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    good = bool(torch.equal(mc, c0) and torch.equal(ml, l0))
    print(f"shard merge (2 x 32 per query) == full-bank top-k: {'ok' if good else 'MISMATCH'}")
    ok &= good
    # k_refresh (cross-multiplied minimum) on 512-bin laws vs the oracle
    rng = np.random.default_rng(5)
    nl, P = 500, 512
    lensr = np.clip(np.round(np.exp(5.5 + 0.8 * rng.standard_normal((nl, 64)))), 1, 2048).astype(np.int64)
    Ir = rng.integers(1, 4097, nl).astype(np.int32)
    gr = np.where(rng.random(nl) < 0.4, rng.integers(0, 2049, nl), 0).astype(np.int32)
    npts = np.zeros(nl, np.int32)
    pc = np.zeros((nl, P), np.int32)
    pD = np.zeros((nl, P), np.int64)
    for i in range(nl):
        v, cnt = np.unique(lensr[i], return_counts=True)
        npts[i] = v.size
        pc[i, :v.size] = cnt
        pD[i, :v.size] = cnt * (v * v + 2 * int(Ir[i]) * v)
    dG = torch.zeros(nl, dtype=torch.float64, device="cuda")
    dI, dg, dn, dpc, dpD = (torch.as_tensor(x, device="cuda") for x in (Ir, gr, npts, pc, pD))
    db = torch.zeros(nl, dtype=torch.int32, device="cuda")
    _lib.call("ss_refresh", nl, _lib.ptr(dI), _lib.ptr(dg), _lib.ptr(db), 200, _lib.ptr(dn),
              _lib.ptr(dpc), _lib.ptr(dpD), P, _lib.ptr(dG), None, 1, _lib.stream_ptr())
    got = dG.cpu().numpy()
    good = all(got[i] == O.gittins_points(pc[i, :npts[i]], pD[i, :npts[i]], int(Ir[i]), int(gr[i]))
               for i in range(nl))
    print(f"refresh of {nl} 512-bin laws: {'ok' if good else 'MISMATCH'}")
    ok &= good
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

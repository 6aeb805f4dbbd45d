"""Trace replay driver for BASELINE configs[4]: rolling bank inserts with a
scheduling round per step.

This is the thin caller the hot path needs to run continuously -- not the
reference's discrete-event engine (out of scope).  Each
round:
  1. the next ``arrivals_per_round`` requests of the trace are admitted:
     predict -> cost -> Gittins on the GPU (SageScheduler.admit), their laws
     stored in the device RequestTable;
  2. every request that ran in the previous round generated
     ``tokens_per_round`` tokens; those that reached their true output length
     complete and their (embedding, length) are pushed into the history ring
     (evicting the oldest);
  3. running requests crossing a 200-token bucket boundary are re-indexed
     (SageScheduler.refresh);
  4. all active requests are ranked (ascending G, id) and the batch for the
     next round is packed on the device over the ranked list (SPEC.md:470
     step 3: projected KV tokens I + g + 1 <= ``kv_capacity``, count <=
     ``batch_size``; ``kv_capacity=None`` keeps only the count limit).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .history import HistoryWindow
from .scheduler import BatchPlan, RequestTable, RoundConfig, SageScheduler, pack_batch, rank

__all__ = ["Trace", "ReplayStats", "replay"]


@dataclass
class Trace:
    """Arrival-ordered requests (ids are the arrival order)."""

    emb: np.ndarray        # int8 [n, dim]
    inv: np.ndarray        # f32 [n]
    input_len: np.ndarray  # int32 [n]
    true_len: np.ndarray   # int32 [n]  realised output length O*


@dataclass
class ReplayStats:
    rounds: int = 0
    admitted: int = 0
    completed: int = 0
    refreshed: int = 0
    fallbacks: int = 0


def replay(window: HistoryWindow, trace: Trace, cfg: RoundConfig, arrivals_per_round: int,
           tokens_per_round: int, batch_size: int, max_active: int, rounds: int,
           on_round=None, kv_capacity: int | None = None, pack_mode: str = "cut") -> ReplayStats:
    """Run ``rounds`` scheduling rounds over ``trace``; ``on_round(r, info)`` sees
    each round's device state (for parity checks)."""
    dev = "cuda"
    sched = SageScheduler(window, cfg)
    table = RequestTable(max_active, cfg.nbins)
    free = list(range(max_active - 1, -1, -1))
    row_of: dict[int, int] = {}
    g_host = np.zeros(max_active, np.int32)
    running: list[int] = []          # request ids that run this round
    nxt = 0
    st = ReplayStats()
    plan = BatchPlan(batch_size)
    K = (1 << 62) if kv_capacity is None else int(kv_capacity)
    for r in range(rounds):
        # 2. progress + completions of the requests that ran last round
        done = []
        for rid in running:
            row = row_of[rid]
            g_host[row] += tokens_per_round
            if g_host[row] >= trace.true_len[rid]:
                done.append(rid)
        if done:
            d = np.array(done)
            window.push(trace.emb[d], trace.true_len[d], trace.inv[d])
            for rid in done:
                free.append(row_of.pop(rid))
            st.completed += len(done)
        # 1. admissions
        n_new = min(arrivals_per_round, trace.emb.shape[0] - nxt, len(free))
        new_ids = np.arange(nxt, nxt + n_new)
        nxt += n_new
        if n_new:
            rows = [free.pop() for _ in range(n_new)]
            for rid, row in zip(new_ids, rows):
                row_of[int(rid)] = row
                g_host[row] = 0
            pst = sched.admit(table, torch.as_tensor(rows, device=dev), trace.emb[new_ids],
                              trace.inv[new_ids], trace.input_len[new_ids], new_ids)
            st.fallbacks += int(pst.used_fb.sum().item())
            st.admitted += n_new
        # 3. refresh of running requests that crossed a bucket boundary
        act_ids = np.array(sorted(row_of), dtype=np.int64)
        act_rows = np.array([row_of[i] for i in act_ids], dtype=np.int64)
        if act_rows.size == 0:
            running = []
            continue
        rows_t = torch.as_tensor(act_rows, device=dev)
        sub = _Sub(table, rows_t)
        g_act = torch.as_tensor(g_host[act_rows], device=dev)
        refreshed = sched.refresh(sub, act_rows.size, g_act)
        sub.write_back(table, rows_t)
        st.refreshed += int(refreshed.sum().item())
        # 4. rank every active request, run the first batch_size
        perm_t = rank(sub.G[:act_rows.size], sub.ids[:act_rows.size])
        pack_batch(perm_t, sub.I[:act_rows.size], g_act, K, batch_size, pack_mode, out=plan)
        batch, _ = plan.host()
        running = [int(act_ids[b]) for b in batch]
        if on_round is not None:
            on_round(r, dict(active_ids=act_ids, G=sub.G.cpu().numpy(), perm=perm_t.cpu().numpy(),
                             g=g_host[act_rows].copy(), running=running))
        st.rounds += 1
    return st


class _Sub:
    """A packed copy of the active rows of the RequestTable (gather / scatter)."""

    def __init__(self, t: RequestTable, rows: torch.Tensor):
        self.P = t.P
        self.I = t.I[rows].contiguous()
        self.g = t.g[rows].contiguous()
        self.bucket = t.bucket[rows].contiguous()
        self.npts = t.npts[rows].contiguous()
        self.ids = t.ids[rows].contiguous()
        self.G = t.G[rows].contiguous()
        self.pcnt = t.pcnt[rows].contiguous()
        self.pD = t.pD[rows].contiguous()

    def write_back(self, t: RequestTable, rows: torch.Tensor):
        t.g[rows] = self.g
        t.bucket[rows] = self.bucket
        t.G[rows] = self.G

"""Device-resident trace replay (BASELINE configs[4]).

The same round as ``replay.replay`` -- completions pushed into the history
ring, admissions predicted, bucket refreshes, full re-rank, batch packed --
with every per-request array kept on the GPU:

  * the active requests live in a RequestTable compacted in increasing id
    order (arrivals are appended with larger ids, completions removed by a
    stable compaction), so rows [0, n_active) are directly the rank input
    and ids double as the SPEC.md:394 arrival tie-break;
  * the running batch is carried as request ids in priority (batch) order,
    which is also the order completions are pushed into the FIFO ring
    (SPEC.md:122-130), exactly as the host driver does;
  * admissions run the fused round entry point (``ss_schedule_round``:
    similarity + merge + histogram + cost + Gittins) writing straight into
    the appended table rows;
  * the batch is carried as a fixed-size id array plus a device count, and
    the statistics stay on the device, so the host learns one number per
    round -- the completion count, which sizes the ring push and the
    compaction.

``tests/test_gpu_parity.py`` checks it round by round against
``replay.replay`` (itself checked against an independent numpy replica).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .history import HistoryWindow
from .replay import ReplayStats, Trace
from .scheduler import BatchPlan, RequestTable, RoundConfig, SageScheduler, pack_batch, rank

__all__ = ["DeviceTrace", "DeviceReplay"]


@dataclass
class DeviceTrace:
    """Arrival-ordered requests on the device (ids are the arrival order)."""

    emb: torch.Tensor        # int8 [n, dim]
    inv: torch.Tensor        # f32 [n]
    input_len: torch.Tensor  # int32 [n]
    true_len: torch.Tensor   # int32 [n]

    @staticmethod
    def from_host(t: Trace) -> "DeviceTrace":
        d = "cuda"
        return DeviceTrace(torch.as_tensor(t.emb, device=d), torch.as_tensor(t.inv, device=d),
                           torch.as_tensor(t.input_len, device=d),
                           torch.as_tensor(t.true_len, device=d))

    def __len__(self):
        return self.emb.shape[0]


class DeviceReplay:
    """Round-by-round replay of ``trace`` against ``window`` on one GPU."""

    def __init__(self, window: HistoryWindow, trace: DeviceTrace, cfg: RoundConfig,
                 arrivals_per_round: int, tokens_per_round: int, batch_size: int,
                 max_active: int, kv_capacity: int | None = None, pack_mode: str = "cut"):
        self.window, self.trace, self.cfg = window, trace, cfg
        self.A, self.TOK, self.B = int(arrivals_per_round), int(tokens_per_round), int(batch_size)
        self.max_active = int(max_active)
        self.K = (1 << 62) if kv_capacity is None else int(kv_capacity)
        self.mode = pack_mode
        self.sched = SageScheduler(window, cfg)
        self.table = RequestTable(self.max_active, cfg.nbins)
        self.plan = BatchPlan(self.B)
        self.n_act = 0
        self.nxt = 0
        # last batch: request ids in priority order, valid below plan.count
        self.run_ids = torch.zeros(self.B, dtype=torch.int64, device="cuda")
        self.plan.count.zero_()
        self.lane = torch.arange(self.B, dtype=torch.int32, device="cuda")
        # device-side counters: completed, refreshed, fallbacks, rounds
        self._dstats = torch.zeros(4, dtype=torch.int64, device="cuda")
        self._admitted = 0
        self._scratch = None
        self._cols = ("I", "g", "bucket", "npts", "ids", "G", "pbin", "pcnt", "pD")

    def _compact(self, keep_rows: torch.Tensor):
        t = self.table
        m = keep_rows.numel()
        for name in self._cols:
            a = getattr(t, name)
            a[:m] = a[keep_rows]
        self.n_act = m

    @property
    def stats(self) -> ReplayStats:
        c, r, f, n = (int(x) for x in self._dstats.tolist())
        return ReplayStats(rounds=n, admitted=self._admitted, completed=c, refreshed=r, fallbacks=f)

    def round(self) -> dict:
        t, tr, n = self.table, self.trace, self.n_act
        # 1. progress of last round's batch; completions enter the ring in
        #    batch order (entries past plan.count are padding, masked out)
        if n:
            valid = self.lane < self.plan.count
            rows = torch.searchsorted(t.ids[:n], self.run_ids).clamp_(max=n - 1)
            t.g.index_add_(0, rows, valid.to(torch.int32) * self.TOK)
            done = valid & (t.g[rows] >= tr.true_len[self.run_ids])
            done_ids = self.run_ids[done]
            nd = done_ids.numel()  # the one host sync of the round: push size
            if nd:
                self.window.push(tr.emb[done_ids], tr.true_len[done_ids], tr.inv[done_ids])
                keep = torch.ones(n, dtype=torch.bool, device="cuda")
                keep[rows[done]] = False
                self._compact(keep.nonzero().squeeze(1))
                self._dstats[0] += nd
        # 2. admissions, appended after the survivors (larger ids: order kept),
        #    predicted by the fused round straight into the table rows
        n = self.n_act
        n_new = min(self.A, len(tr) - self.nxt, self.max_active - n)
        if n_new > 0:
            lo, c = self.nxt, self.cfg
            t.ids[n:n + n_new] = torch.arange(lo, lo + n_new, dtype=torch.int64, device="cuda")
            t.I[n:n + n_new] = tr.input_len[lo:lo + n_new]
            t.g[n:n + n_new] = 0
            t.bucket[n:n + n_new] = 0
            if self._scratch is None or self._scratch[0].numel() < n_new:
                self._scratch = (torch.empty(n_new, dtype=torch.int64, device="cuda"),
                                 torch.empty(n_new, dtype=torch.uint8, device="cuda"))
            perm_s, fb = self._scratch
            _lib.call("ss_schedule_round", self.window.handle, _lib.ptr(tr.emb[lo:lo + n_new]),
                      _lib.ptr(tr.inv[lo:lo + n_new]), _lib.ptr(t.I[n:]), _lib.ptr(t.ids[n:]),
                      n_new, c.k, float(np.float32(c.theta)), c.min_matches, c.max_len, c.nbins,
                      _lib.ALGO[c.algo], t.P, _lib.ptr(t.npts[n:]), _lib.ptr(t.pbin[n:]),
                      _lib.ptr(t.pcnt[n:]), _lib.ptr(t.pD[n:]), _lib.ptr(fb), _lib.ptr(t.G[n:]),
                      _lib.ptr(perm_s), _lib.stream_ptr())
            self._dstats[2] += fb[:n_new].sum()
            self._admitted += n_new
            self.nxt += n_new
            self.n_act = n = n + n_new
        if n == 0:
            self.plan.count.zero_()
            return dict(perm=torch.zeros(0, dtype=torch.int64, device="cuda"), n_active=0)
        # 3. bucket refreshes of requests whose progress crossed a boundary
        refreshed = self.sched.refresh(t, n, t.g[:n])
        self._dstats[1] += refreshed.sum()
        # 4. rank and pack the next batch on the device
        perm = rank(t.G[:n], t.ids[:n])
        pack_batch(perm, t.I[:n], t.g[:n], self.K, self.B, self.mode, out=self.plan)
        self.run_ids = t.ids[:n][self.plan.batch.clamp(0, n - 1)]
        self._dstats[3] += 1
        return dict(perm=perm, n_active=n)

    def running(self) -> list:
        cnt = int(self.plan.count.item())
        if cnt < 0:
            raise ValueError("request cannot fit: I + 1 exceeds the KV capacity")
        return self.run_ids[:cnt].cpu().tolist()

    def info(self, perm) -> dict:
        """Host copy of the round's state, in replay.replay's on_round format."""
        n = self.n_act
        return dict(active_ids=self.table.ids[:n].cpu().numpy(), G=self.table.G[:n].cpu().numpy(),
                    perm=perm.cpu().numpy(), running=self.running())


class NativeReplay:
    """The same replay with each round a single C-ABI call (``ss_engine_round``,
    csrc/k_engine.cu): progress, ring push, compaction, admission, refresh,
    rank and packing all launched natively from one host call."""

    def __init__(self, window: HistoryWindow, trace: DeviceTrace, cfg: RoundConfig,
                 arrivals_per_round: int, tokens_per_round: int, batch_size: int,
                 max_active: int, kv_capacity: int | None = None, pack_mode: str = "cut"):
        import ctypes as C

        from .scheduler import PACK_MODE

        self._C = C
        self.window, self.trace, self.cfg = window, trace, cfg
        self.A, self.TOK, self.B = int(arrivals_per_round), int(tokens_per_round), int(batch_size)
        self.K = (1 << 62) if kv_capacity is None else int(kv_capacity)
        self.mode = PACK_MODE[pack_mode]
        h = C.c_void_p()
        _lib.call("ss_table_create", C.byref(h), torch.cuda.current_device(), int(max_active),
                  cfg.nbins, self.B)
        self._t = h
        self._next = C.c_int64(0)
        self.stats = ReplayStats()

    def close(self):
        if getattr(self, "_t", None) is not None and self._t.value:
            _lib.lib().ss_table_destroy(self._t)
            self._t = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def round(self) -> dict:
        C, c, tr = self._C, self.cfg, self.trace
        nd, na = C.c_int64(0), C.c_int64(0)
        _lib.call("ss_engine_round", self._t, self.window.handle, _lib.ptr(tr.emb), _lib.ptr(tr.inv),
                  _lib.ptr(tr.input_len), _lib.ptr(tr.true_len), len(tr), C.byref(self._next),
                  self.A, self.TOK, c.bucket_size, self.K, self.mode, c.k,
                  float(np.float32(c.theta)), c.min_matches, c.max_len, c.nbins, _lib.ALGO[c.algo],
                  C.byref(nd), C.byref(na), _lib.stream_ptr())
        self.stats.completed += nd.value
        self.stats.admitted += na.value
        n = self.n_act
        if n:
            self.stats.rounds += 1
        return dict(n_active=n)

    def _view(self):
        C = self._C
        n = C.c_int64(0)
        ptrs = [C.c_void_p() for _ in range(8)]
        _lib.call("ss_table_view", self._t, C.byref(n), *[C.byref(p) for p in ptrs])
        return n.value, [p.value for p in ptrs]

    @property
    def n_act(self) -> int:
        return self._view()[0]

    def info(self, _=None) -> dict:
        """Host copy of the round's state, in replay.replay's on_round format."""
        from .history import _cuda_view

        n, (pI, pg, pids, pG, pnp, pperm, prun, pcnt) = self._view()
        dev = torch.cuda.current_device()
        ids = _cuda_view(pids, torch.int64, (n,), dev).cpu().numpy()
        G = _cuda_view(pG, torch.float64, (n,), dev).cpu().numpy()
        perm = _cuda_view(pperm, torch.int64, (n,), dev).cpu().numpy()
        cnt = int(_cuda_view(pcnt, torch.int32, (1,), dev).item())
        if cnt < 0:
            raise ValueError("request cannot fit: I + 1 exceeds the KV capacity")
        run = _cuda_view(prun, torch.int64, (self.B,), dev)[:cnt].cpu().tolist()
        return dict(active_ids=ids, G=G, perm=perm, running=run)

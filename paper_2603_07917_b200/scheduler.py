"""The per-round scheduling hot path, batched on the GPU.

    predict  (stage 1+1b)  ss_topk -> window fallback histogram -> ss_finish
    cost     (stage 2)     fused in ss_finish (ResourceBound, cost.py:97-99)
    Gittins  (stage 3)     fused in ss_finish; ss_refresh for running requests
    rank     (stage 4)     ss_rank, ascending (G, id)

``SageScheduler`` is what an engine loop calls once per
iteration: ``admit`` runs predict+cost+Gittins for newly arrived requests,
``refresh`` re-indexes running requests that crossed a bucket boundary, and
``rank`` orders every active request.  ``schedule_round`` is the fused single
call for a batch of pending requests (the bench workload), and
``schedule_round_host`` the same from host buffers (the plugin call).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .history import HistoryWindow, _as_vectors, split_wide

__all__ = ["BatchPlan", "pack_batch", "RoundConfig", "PredictState", "RequestTable", "SageScheduler", "rank"]


@dataclass(frozen=True)
class RoundConfig:
    k: int = 64
    theta: float = 0.8
    min_matches: int = 20
    max_len: int = 2048         # O_max
    nbins: int = 128
    bucket_size: int = 200
    algo: str = "auto"

    def __post_init__(self):
        if not 1 <= self.k <= 256:
            raise ValueError("k must lie in [1, 256]")
        if self.max_len % self.nbins:
            raise ValueError("max_len must be a multiple of nbins")
        if not -1.0 <= self.theta <= 1.0:
            raise ValueError("theta must lie in [-1, 1]")


@dataclass
class PredictState:
    """Device outputs of stages 1-3 for a batch of requests."""

    comp: torch.Tensor    # int64 [n, k] neighbour composites (desc), 0 = none
    nbr_len: torch.Tensor  # int32 [n, k]
    npts: torch.Tensor    # int32 [n]
    pbin: torch.Tensor    # int32 [n, P]
    pcnt: torch.Tensor    # int32 [n, P]
    pD: torch.Tensor      # int64 [n, P]  sum v^2 + 2 I sum v per bin
    psv: torch.Tensor     # int64 [n, P]  sum v per bin
    used_fb: torch.Tensor  # uint8 [n]
    G: torch.Tensor       # float64 [n]

    def cost_law(self, i: int):
        """(support, masses) of request i's cost law on the host."""
        n = int(self.npts[i].item())
        c = self.pcnt[i, :n].double()
        D = self.pD[i, :n].double()
        s = (D * 0.5) / c
        return s.cpu().numpy(), (c / c.sum()).cpu().numpy()


def rank(G: torch.Tensor, ids: torch.Tensor | None = None, perm: torch.Tensor | None = None,
         workspace: torch.Tensor | None = None) -> torch.Tensor:
    """Indices ordering requests by ascending (G, id)."""
    n = G.numel()
    if perm is None:
        perm = torch.empty(n, dtype=torch.int64, device=G.device)
    wsb = int(_lib.lib().ss_rank_workspace_bytes(n))
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty(wsb, dtype=torch.uint8, device=G.device)
    _lib.call("ss_rank", _lib.ptr(G), _lib.ptr(ids), n, _lib.ptr(perm), _lib.ptr(workspace), wsb,
              _lib.stream_ptr())
    return perm


PACK_MODE = {"cut": 0, "skip": 1}


class BatchPlan:
    """Device result of ``pack_batch``: ``batch[:count]`` request indices in
    priority order, projecting ``tokens`` KV tokens."""

    def __init__(self, max_batch: int, device="cuda"):
        self.batch = torch.empty(max_batch, dtype=torch.int64, device=device)
        self.count = torch.zeros(1, dtype=torch.int32, device=device)
        self.tokens = torch.zeros(1, dtype=torch.int64, device=device)

    def host(self):
        """(batch int64 [count] numpy, tokens) after a synchronising read;
        raises ValueError for a request that can never fit (SPEC.md engine
        step errors: "request cannot fit")."""
        n = int(self.count.item())
        t = int(self.tokens.item())
        if n < 0:
            raise ValueError(f"request {t} cannot fit: I + 1 exceeds the KV capacity")
        return self.batch[:n].cpu().numpy(), t


def pack_batch(perm: torch.Tensor, input_len: torch.Tensor, g: torch.Tensor,
               kv_capacity: int = 8192, max_batch: int = 64, mode: str = "cut",
               out: BatchPlan | None = None, stream=None) -> BatchPlan:
    """Engine batch formation over the ranked list (SPEC.md:470 step 3,
    defaults K = 8192, B = 64 from SPEC.md:501): admit requests in ``perm``
    order while sum(I + g + 1) <= K and count <= B.  ``mode`` "cut" stops at
    the first request that does not fit, "skip" passes over it.  Async on the
    device (graph-capturable); ``BatchPlan.host()`` reads the result."""
    if mode not in PACK_MODE:
        raise ValueError(f"mode must be one of {sorted(PACK_MODE)}, got {mode!r}")
    n = perm.numel()
    if out is None:
        out = BatchPlan(max_batch, perm.device)
    elif out.batch.numel() < max_batch:
        raise ValueError("BatchPlan smaller than max_batch")
    _lib.call("ss_pack_batch", _lib.ptr(perm), _lib.ptr(input_len), _lib.ptr(g), n,
              int(kv_capacity), int(max_batch), PACK_MODE[mode], _lib.ptr(out.batch),
              _lib.ptr(out.count), _lib.ptr(out.tokens), _lib.stream_ptr(stream))
    return out


class RequestTable:
    """Device-resident per-request state for active (pending+running) requests.

    HBM layout, one row per request slot:
      I, g, bucket, npts int32 [cap]; ids int64 [cap]; G float64 [cap]
      pcnt int32 [cap, P], pD int64 [cap, P] -- the sparse cost law
    """

    def __init__(self, capacity: int, P: int):
        dev = "cuda"
        self.capacity, self.P = int(capacity), int(P)
        self.I = torch.zeros(capacity, dtype=torch.int32, device=dev)
        self.g = torch.zeros(capacity, dtype=torch.int32, device=dev)
        self.bucket = torch.zeros(capacity, dtype=torch.int32, device=dev)
        self.npts = torch.zeros(capacity, dtype=torch.int32, device=dev)
        self.ids = torch.zeros(capacity, dtype=torch.int64, device=dev)
        self.G = torch.full((capacity,), float("inf"), dtype=torch.float64, device=dev)
        self.pbin = torch.zeros((capacity, P), dtype=torch.int32, device=dev)
        self.pcnt = torch.zeros((capacity, P), dtype=torch.int32, device=dev)
        self.pD = torch.zeros((capacity, P), dtype=torch.int64, device=dev)


class SageScheduler:
    """Batched SageSched scheduling on one GPU's history window."""

    def __init__(self, window: HistoryWindow, cfg: RoundConfig = RoundConfig()):
        _lib.require_cuda()
        self.window = window
        self.cfg = cfg
        self.fallback_events = 0  # SPEC.md:194 fallback counter
        self._host_call = None  # cached ss_schedule_round_host arguments

    # ---------------------------------------------------------- stages 1-3 --
    def predict(self, q, q_inv, input_len, stream=None) -> PredictState:
        c = self.cfg
        q = _as_vectors(q)  # int8, or int16 exact counts (wide pass)
        q_inv = torch.as_tensor(q_inv, device="cuda").to(torch.float32).contiguous()
        I = torch.as_tensor(input_len, device="cuda").to(torch.int32).contiguous()
        if len(self.window) == 0:
            raise _lib.ColdStartError("cold start: the history window is empty (SPEC.md:190)")
        n = q.shape[0]
        comp, ln = self.window.topk(q, q_inv, c.k, c.theta, c.algo, stream)
        fb = self.window.fallback_hist(c.max_len, c.nbins, stream)
        P = c.nbins
        st = PredictState(
            comp=comp, nbr_len=ln,
            npts=torch.zeros(n, dtype=torch.int32, device="cuda"),
            pbin=torch.zeros((n, P), dtype=torch.int32, device="cuda"),
            pcnt=torch.zeros((n, P), dtype=torch.int32, device="cuda"),
            pD=torch.zeros((n, P), dtype=torch.int64, device="cuda"),
            psv=torch.zeros((n, P), dtype=torch.int64, device="cuda"),
            used_fb=torch.zeros(n, dtype=torch.uint8, device="cuda"),
            G=torch.empty(n, dtype=torch.float64, device="cuda"))
        _lib.call("ss_finish", _lib.ptr(comp), _lib.ptr(ln), n, c.k, c.min_matches, c.max_len,
                  c.nbins, _lib.ptr(I), _lib.ptr(fb[0]), _lib.ptr(fb[1]), _lib.ptr(fb[2]), P,
                  _lib.ptr(st.npts), _lib.ptr(st.pbin), _lib.ptr(st.pcnt), _lib.ptr(st.pD),
                  _lib.ptr(st.psv), _lib.ptr(st.used_fb), _lib.ptr(st.G), _lib.stream_ptr(stream))
        return st

    def admit(self, table: RequestTable, rows: torch.Tensor, q, q_inv, input_len, ids,
              stream=None) -> PredictState:
        """Predict for newly admitted requests and store their laws in `table`."""
        st = self.predict(q, q_inv, input_len, stream)
        rows = rows.to(device="cuda", dtype=torch.int64)
        P = min(table.P, st.pcnt.shape[1])
        table.I[rows] = torch.as_tensor(input_len, device="cuda").to(torch.int32)
        table.g[rows] = 0
        table.bucket[rows] = 0
        table.ids[rows] = torch.as_tensor(ids, device="cuda").to(torch.int64)
        table.npts[rows] = st.npts
        table.pbin[rows, :P] = st.pbin[:, :P]
        table.pcnt[rows, :P] = st.pcnt[:, :P]
        table.pD[rows, :P] = st.pD[:, :P]
        table.G[rows] = st.G
        self.fallback_events += int(st.used_fb.sum().item())
        return st

    def refresh(self, table: RequestTable, n: int, g_new: torch.Tensor, force: bool = False,
                stream=None) -> torch.Tensor:
        """Re-index rows [0, n) that crossed a bucket boundary."""
        table.g[:n] = g_new.to(device="cuda", dtype=torch.int32)
        refreshed = torch.zeros(n, dtype=torch.uint8, device="cuda")
        _lib.call("ss_refresh", n, _lib.ptr(table.I), _lib.ptr(table.g), _lib.ptr(table.bucket),
                  self.cfg.bucket_size, _lib.ptr(table.npts), _lib.ptr(table.pcnt),
                  _lib.ptr(table.pD), table.P, _lib.ptr(table.G), _lib.ptr(refreshed),
                  1 if force else 0, _lib.stream_ptr(stream))
        return refreshed

    def rank(self, table: RequestTable, n: int) -> torch.Tensor:
        return rank(table.G[:n], table.ids[:n])

    # ------------------------------------------------------------ fused -----
    def schedule_round(self, q, q_inv, input_len, ids=None, out=None, stream=None):
        """One fused round for a batch of pending requests (device tensors).

        Returns (perm int64 [n], G float64 [n], PredictState-like buffers).
        int16 queries (exact feature-hash counts beyond int8) run the wide
        pass for the rows that need it (ss_schedule_round_wide)."""
        c = self.cfg
        n = q.shape[0]
        if out is None:
            out = self.round_buffers(n)
        if q.dtype != torch.int8:
            q8, qi, widx, wq, winv = split_wide(_as_vectors(q), q_inv)
            if widx is not None:
                _lib.call("ss_schedule_round_wide", self.window.handle, _lib.ptr(q8), _lib.ptr(qi),
                          _lib.ptr(input_len), _lib.ptr(ids), n, widx.numel(), _lib.ptr(widx),
                          _lib.ptr(wq), _lib.ptr(winv), c.k, float(np.float32(c.theta)),
                          c.min_matches, c.max_len, c.nbins, _lib.ALGO[c.algo], c.nbins,
                          _lib.ptr(out["npts"]), _lib.ptr(out["pbin"]), _lib.ptr(out["pcnt"]),
                          _lib.ptr(out["pD"]), _lib.ptr(out["used_fb"]), _lib.ptr(out["G"]),
                          _lib.ptr(out["perm"]), _lib.stream_ptr(stream))
                return out["perm"], out["G"], out
            q = q8
        _lib.call("ss_schedule_round", self.window.handle, _lib.ptr(q), _lib.ptr(q_inv),
                  _lib.ptr(input_len), _lib.ptr(ids), n, c.k, float(np.float32(c.theta)),
                  c.min_matches, c.max_len, c.nbins, _lib.ALGO[c.algo], c.nbins,
                  _lib.ptr(out["npts"]), _lib.ptr(out["pbin"]), _lib.ptr(out["pcnt"]),
                  _lib.ptr(out["pD"]), _lib.ptr(out["used_fb"]), _lib.ptr(out["G"]),
                  _lib.ptr(out["perm"]), _lib.stream_ptr(stream))
        return out["perm"], out["G"], out

    def round_buffers(self, n: int):
        P = self.cfg.nbins
        d = "cuda"
        return dict(npts=torch.zeros(n, dtype=torch.int32, device=d),
                    pbin=torch.zeros((n, P), dtype=torch.int32, device=d),
                    pcnt=torch.zeros((n, P), dtype=torch.int32, device=d),
                    pD=torch.zeros((n, P), dtype=torch.int64, device=d),
                    used_fb=torch.zeros(n, dtype=torch.uint8, device=d),
                    G=torch.zeros(n, dtype=torch.float64, device=d),
                    perm=torch.zeros(n, dtype=torch.int64, device=d))

    def schedule_round_host(self, q: np.ndarray, q_inv: np.ndarray, input_len: np.ndarray,
                            ids: np.ndarray | None = None, G_out: np.ndarray | None = None,
                            perm_out: np.ndarray | None = None, stream=None):
        """The plugin call from host buffers: H2D, round, D2H, synchronise."""
        c = self.cfg
        n = q.shape[0]
        if G_out is None:
            G_out = np.empty(n, dtype=np.float64)
        if perm_out is None:
            perm_out = np.empty(n, dtype=np.int64)

        # the engine calls this once per iteration with the same buffers: the
        # argument tuple is rebuilt only when a buffer object, the stream or
        # the config changes (numpy arrays never move their data)
        bufs = (q, q_inv, input_len, ids, G_out, perm_out)
        sp = _lib.stream_ptr(stream)
        key = (n, c.k, c.theta, c.min_matches, c.max_len, c.nbins, c.algo)
        hc = self._host_call
        if (hc is None or hc[2] != sp or hc[3] != key or hc[4] != self.window.handle
                or any(x is not y for x, y in zip(bufs, hc[0]))):
            # the C ABI reads raw pointers: check each buffer's dtype, layout
            # and length once per argument tuple (a silent mismatch, e.g. an
            # int64 input_len, would otherwise be read as wrong values)
            dim = self.window.dim
            want = (("q", q, np.int8, (n, dim)), ("q_inv", q_inv, np.float32, (n,)),
                    ("input_len", input_len, np.int32, (n,)), ("ids", ids, np.int64, (n,)),
                    ("G_out", G_out, np.float64, (n,)), ("perm_out", perm_out, np.int64, (n,)))
            for name, a, dt, shape in want:
                if a is None and name == "ids":
                    continue
                if not isinstance(a, np.ndarray):
                    raise TypeError(f"{name} must be a numpy array, got {type(a).__name__}")
                if a.dtype != dt or tuple(a.shape) != shape or not a.flags["C_CONTIGUOUS"]:
                    raise ValueError(f"{name}: need a C-contiguous {np.dtype(dt).name} array of shape "
                                     f"{shape}, got {a.dtype} {tuple(a.shape)}"
                                     f"{'' if a.flags['C_CONTIGUOUS'] else ' (not contiguous)'}")
                if name in ("G_out", "perm_out") and not a.flags["WRITEABLE"]:
                    raise ValueError(f"{name} must be writeable")

            def hp(a):
                return None if a is None else a.ctypes.data

            args = (self.window.handle, hp(q), hp(q_inv), hp(input_len), hp(ids), n, c.k,
                    float(np.float32(c.theta)), c.min_matches, c.max_len, c.nbins,
                    _lib.ALGO[c.algo], hp(G_out), hp(perm_out), sp)
            hc = self._host_call = (bufs, args, sp, key, self.window.handle)
        rc = _lib.lib().ss_schedule_round_host(*hc[1])
        if rc:
            _lib.check(rc, "ss_schedule_round_host")
        return perm_out, G_out

    def capture_round(self, q, q_inv, input_len, ids=None, warmup: int = 2):
        """CUDA-graph the fused round for fixed input buffers; returns (graph, out)."""
        out = self.round_buffers(q.shape[0])
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.schedule_round(q, q_inv, input_len, ids, out, stream=s)
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.schedule_round(q, q_inv, input_len, ids, out)
        return g, out

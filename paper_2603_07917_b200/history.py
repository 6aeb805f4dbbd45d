"""GPU-resident history window (embedding_history module).

A bounded FIFO ring of records (int8 embedding, fp32 inverse norm, realised
output length, insertion_seq), owned by libsagesched (``ss_bank_*``) and
laid out in HBM as

    emb  int8  [capacity, dim]   row-major, 16-byte aligned rows (TMA tiles)
    inv  fp32  [capacity]        1/||emb||, NaN for empty or zero rows
    lens int32 [capacity]
    seq  int64 [capacity]        -1 = empty slot

plus, once a row outside the int8 range is pushed (a long prompt whose
feature-hash bucket exceeds 127, _kernels.py:82-95), a wide plane: the exact
int16 vector and inverse norm of such rows per slot, scored exactly by the
library's CUDA-core wide pass (its int8 row is zero with a NaN norm).

slot = insertion_seq mod capacity, so pushing evicts the oldest record
(SPEC.md:122-130).  Embeddings are the reference's integer feature-hash
vectors kept unnormalised (_kernels.py:64-65), with the L2 normalisation
 carried by ``inv`` -- cosine = dot * inv_q * inv_w.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

__all__ = ["HistoryRecord", "HistoryWindow", "embed", "embed_batch", "push", "query_similar",
           "DEFAULT_SALT"]

DEFAULT_SALT = 0x5A6E5C4E  # fixed feature-hash salt ("with a fixed salt")


@dataclass(frozen=True)
class HistoryRecord:
    embedding: np.ndarray  # int8 [dim]
    realized_output_len: int
    insertion_seq: int


def _as_dev(x, dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda").to(dtype).contiguous()


def _as_vectors(x) -> torch.Tensor:
    """Integer embedding rows on the device: int8 stays int8; any other integer
    dtype becomes int16 (the exact feature-hash counts, |x| <= 32767)."""
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(x))
    if t.is_floating_point():
        raise TypeError(f"embeddings must be integer vectors, got {t.dtype}")
    if t.dtype == torch.int8:
        return t.to("cuda").contiguous()
    t = t.to("cuda")
    if t.numel() and int(t.abs().max().item()) > 32767:
        raise ValueError("an embedding bucket exceeds the int16 range (|x| > 32767)")
    return t.to(torch.int16).contiguous()


def split_wide(q: torch.Tensor, q_inv: torch.Tensor):
    """int16 query rows -> (int8 stand-ins, q_inv, wide index, wide int16 rows,
    wide inverse norms); rows that fit int8 are exact in the stand-ins, the
    others are scored from their int16 vectors by the wide pass."""
    wide = (q.abs() > 127).any(dim=1)
    idx = torch.nonzero(wide).flatten()
    q8 = q.clamp(-127, 127).to(torch.int8).contiguous()
    if idx.numel() == 0:
        return q8, q_inv, None, None, None
    return (q8, q_inv, idx.to(torch.int64).contiguous(), q[idx].contiguous(),
            q_inv[idx].contiguous())


class HistoryWindow:
    """FIFO history bank on one GPU (or one shard of a sharded ring)."""

    def __init__(self, capacity: int = 10_000, dim: int = 384, device: int | None = None,
                 global_capacity: int | None = None, slot_offset: int = 0):
        _lib.require_cuda()
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.capacity = int(capacity)
        self.dim = int(dim)
        self.global_capacity = int(global_capacity or capacity)
        self.slot_offset = int(slot_offset)
        h = C.c_void_p()
        _lib.call("ss_bank_create", C.byref(h), self.device, self.capacity, self.dim,
                  self.global_capacity, self.slot_offset)
        self._h = h

    # -- lifecycle ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.lib().ss_bank_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- state ---------------------------------------------------------------
    def info(self):
        head, size, cap = C.c_int64(), C.c_int64(), C.c_int64()
        dim = C.c_int32()
        _lib.call("ss_bank_info", self._h, C.byref(head), C.byref(size), C.byref(cap), C.byref(dim))
        return int(head.value), int(size.value)

    @property
    def head(self) -> int:
        return self.info()[0]

    def __len__(self) -> int:
        return self.info()[1]

    def tensors(self):
        """Zero-copy views of the device arrays (emb, inv, lens, seq)."""
        e, i, l, s = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.call("ss_bank_device_ptrs", self._h, C.byref(e), C.byref(i), C.byref(l), C.byref(s))
        n = self.capacity

        def view(p, dtype, shape):
            return _cuda_view(p.value, dtype, shape, self.device)

        return (view(e, torch.int8, (n, self.dim)), view(i, torch.float32, (n,)),
                view(l, torch.int32, (n,)), view(s, torch.int64, (n,)))

    # -- mutation ------------------------------------------------------------
    def push(self, emb, lens, inv_norm=None, stream=None) -> None:
        """Append records at the head, evicting the oldest.
        int8 rows enter the tensor-core plane; wider integer rows (int16: the
        exact counts of long prompts) keep their exact vectors when they do
        not fit int8."""
        emb = _as_vectors(emb)
        if emb.dim() == 1:
            emb = emb.reshape(1, -1)
        if emb.shape[1] != self.dim:
            raise ValueError(f"embedding dim {emb.shape[1]} != window dim {self.dim}")
        lens = _as_dev(np.atleast_1d(lens) if not isinstance(lens, torch.Tensor) else lens, torch.int32)
        if lens.numel() != emb.shape[0]:
            raise ValueError("one realised length per record is required")
        inv = None if inv_norm is None else _as_dev(inv_norm, torch.float32)
        st = _lib.stream_ptr(stream)
        _lib.call("ss_bank_push16" if emb.dtype == torch.int16 else "ss_bank_push", self._h,
                  _lib.ptr(emb), _lib.ptr(inv), _lib.ptr(lens), emb.shape[0], st)
        _lib.call("ss_bank_sync_check", self._h, st)

    def write(self, emb, lens, seq, local_slot, inv_norm=None, stream=None) -> None:
        """Scatter records to explicit local slots (sharded ring maintenance)."""
        emb = _as_vectors(emb)
        lens = _as_dev(lens, torch.int32)
        seq = _as_dev(seq, torch.int64)
        slot = _as_dev(local_slot, torch.int64)
        inv = None if inv_norm is None else _as_dev(inv_norm, torch.float32)
        _lib.call("ss_bank_write16" if emb.dtype == torch.int16 else "ss_bank_write", self._h,
                  _lib.ptr(emb), _lib.ptr(inv), _lib.ptr(lens), _lib.ptr(seq), _lib.ptr(slot),
                  emb.shape[0], _lib.stream_ptr(stream))

    def set_head(self, global_head: int) -> None:
        _lib.call("ss_bank_set_head", self._h, int(global_head))

    def fallback_hist(self, max_len: int, nbins: int, stream=None):
        """Window-wide binned length histogram (cnt, sum_v, sum_v2) int64 [nbins]."""
        out = torch.empty((3, nbins), dtype=torch.int64, device="cuda")
        _lib.call("ss_bank_fallback_hist", self._h, int(max_len), int(nbins), _lib.ptr(out[0]),
                  _lib.ptr(out[1]), _lib.ptr(out[2]), _lib.stream_ptr(stream))
        return out

    # -- retrieval -----------------------------------------------------------
    def topk(self, q, q_inv, k: int, theta: float = -1.0, algo: str = "auto", stream=None):
        """Stage 1: per query the top-k rows by (cos desc, seq desc), cos >= theta.

        Returns (comp u64-as-int64 [nq,k], len int32 [nq,k]); see ``decode``.
        Queries may be int16 (exact counts outside int8: the wide pass).
        """
        q = _as_vectors(q)
        q_inv = _as_dev(q_inv, torch.float32)
        nq = q.shape[0]
        comp = torch.zeros((nq, k), dtype=torch.int64, device="cuda")
        ln = torch.zeros((nq, k), dtype=torch.int32, device="cuda")
        if q.dtype == torch.int16:
            q, q_inv, widx, wq, winv = split_wide(q, q_inv)
            if widx is not None:
                _lib.call("ss_topk_wide", self._h, _lib.ptr(q), _lib.ptr(q_inv), nq, widx.numel(),
                          _lib.ptr(widx), _lib.ptr(wq), _lib.ptr(winv), int(k),
                          float(np.float32(theta)), _lib.ALGO[algo], _lib.ptr(comp), _lib.ptr(ln),
                          _lib.stream_ptr(stream))
                return comp, ln
        _lib.call("ss_topk", self._h, _lib.ptr(q), _lib.ptr(q_inv), nq, int(k),
                  float(np.float32(theta)), _lib.ALGO[algo], _lib.ptr(comp), _lib.ptr(ln),
                  _lib.stream_ptr(stream))
        return comp, ln

    def decode(self, comp: torch.Tensor, stream=None):
        """composites -> (cos f32, insertion_seq i64, global slot i64); empty -> (nan,-1,-1)."""
        n = comp.numel()
        key = torch.empty(comp.shape, dtype=torch.float32, device="cuda")
        seq = torch.empty(comp.shape, dtype=torch.int64, device="cuda")
        slot = torch.empty(comp.shape, dtype=torch.int64, device="cuda")
        _lib.call("ss_decode_topk", _lib.ptr(comp), n, self.head, self.global_capacity,
                  _lib.ptr(key), _lib.ptr(seq), _lib.ptr(slot), _lib.stream_ptr(stream))
        return key, seq, slot


def _cuda_view(addr: int, dtype, shape, device: int) -> torch.Tensor:
    """A torch tensor aliasing library-owned device memory (no copy)."""

    class _Iface:
        __cuda_array_interface__ = {
            "shape": tuple(shape),
            "typestr": {torch.int8: "|i1", torch.float32: "<f4", torch.int32: "<i4",
                        torch.int64: "<i8", torch.float64: "<f8"}[dtype],
            "data": (addr, False),
            "version": 3,
            "strides": None,
        }

    return torch.as_tensor(_Iface(), device=f"cuda:{device}")


def embed_batch(prompts, salt: int = DEFAULT_SALT, dim: int = 384):
    """Feature-hash prompts on the device (SPEC.md:112-120 embed; hash of
    _kernels.py:37-102): (exact integer vectors, fp32 inverse norms).  The
    vectors are int8 when every bucket of every prompt fits, else int16 (the
    bank and the round keep such rows exact through the wide pass)."""
    _lib.require_cuda()
    offs = np.zeros(len(prompts) + 1, dtype=np.int64)
    offs[1:] = np.cumsum([len(p) for p in prompts])
    flat = np.concatenate([np.asarray(p, np.int64) for p in prompts]) if offs[-1] else np.zeros(1, np.int64)
    t = torch.as_tensor(flat, device="cuda")
    o = torch.as_tensor(offs, device="cuda")
    n = len(prompts)
    emb = torch.empty((n, dim), dtype=torch.int16, device="cuda")
    inv = torch.empty(n, dtype=torch.float32, device="cuda")
    n_wide = C.c_int64()
    _lib.call("ss_embed_quantize_batch", _lib.ptr(t), _lib.ptr(o), n, int(salt) & (2**64 - 1),
              int(dim), _lib.ptr(emb), _lib.ptr(inv), C.byref(n_wide), _lib.stream_ptr())
    return (emb if n_wide.value else emb.to(torch.int8)), inv


def embed(prompt_tokens, salt: int = DEFAULT_SALT, dim: int = 384):
    """One prompt -> (int8 embedding, inverse norm); empty prompt -> zero vector
    with NaN inverse norm (the SPEC's "degenerate embedding" flag)."""
    e, i = embed_batch([prompt_tokens], salt, dim)
    return e[0], i[0]


def push(window: HistoryWindow, record: HistoryRecord) -> HistoryWindow:
    """SPEC.md:122 push(window, record); insertion_seq is assigned by the ring."""
    e = record.embedding
    e = e.reshape(1, -1) if isinstance(e, torch.Tensor) else np.asarray(e).reshape(1, -1)
    window.push(e, np.array([record.realized_output_len], np.int32))
    return window


def query_similar(window: HistoryWindow, q, q_inv, theta: float):
    """EVERY record with cos >= theta, desc cos, tie -> larger
    insertion_seq (theta = -1 returns the whole window).  One query (its
    exact integer vector, int8 or int16) and its inverse norm.

    Returns (seq int64 [m], cos float32 [m], length int32 [m]) on the host.
    """
    if not -1.0 <= theta <= 1.0:
        raise ValueError(f"theta must lie in [-1, 1], got {theta}")
    q = _as_vectors(q).reshape(-1).to(torch.int16).contiguous()
    if q.numel() != window.dim:
        raise ValueError(f"query dim {q.numel()} != window dim {window.dim}")
    qi = float(q_inv.item() if isinstance(q_inv, torch.Tensor) else np.float32(np.asarray(q_inv).reshape(-1)[0]))
    cap = window.capacity
    key = torch.empty(cap, dtype=torch.float32, device="cuda")
    seq = torch.empty(cap, dtype=torch.int64, device="cuda")
    ln = torch.empty(cap, dtype=torch.int32, device="cuda")
    m = C.c_int64()
    _lib.call("ss_query_similar", window.handle, _lib.ptr(q), qi, float(np.float32(theta)),
              _lib.ptr(key), _lib.ptr(seq), _lib.ptr(ln), C.byref(m), _lib.stream_ptr())
    n = m.value
    return seq[:n].cpu().numpy(), key[:n].cpu().numpy(), ln[:n].cpu().numpy()

"""Drop-in for ``servesim._kernels`` (the reference's plugin boundary).

Same function names, argument meaning and error behaviour as
/root/reference/pkg/src/servesim/_kernels.py, but every call runs a
hand-written sm_100a kernel through libsagesched's C ABI.  There is no
numba/numpy switch (``HAVE_NUMBA`` is gone): a missing library or device
raises instead of falling back.

Arguments may be numpy arrays (host; copied to and from the device, as a
reference caller would pass them) or CUDA torch tensors (used in place).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib

__all__ = ["embed_accumulate", "gittins_min", "match_pmfs", "warmup",
           "gittins_min_batch", "embed_accumulate_batch"]


def _dev(x, dtype) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), device="cuda").to(dtype).contiguous()


def match_pmfs(sims, lens, theta, max_len, sup, mas, sizes) -> None:
    """Threshold match -> exact integer-length pmf (_kernels.py:118-138).

    Writes ``sup[q, :sizes[q]]`` (lengths, ascending), ``mas`` and ``sizes`` in
    place, like the reference.  Masses are bit-identical to the numba path
    (c * (1.0/total)); len == 0 is counted but never emitted.  A matched length
    outside [0, max_len] raises ValueError (undefined behaviour in numba).
    """
    _lib.require_cuda()
    d_sims = _dev(sims, torch.float32)
    nq, nw = d_sims.shape
    d_lens = _dev(lens, torch.int64)
    stride = max(int(sup.shape[1]), int(max_len))
    on_dev = isinstance(sup, torch.Tensor) and sup.is_cuda and sup.shape[1] >= max_len
    d_sup = sup if on_dev else torch.zeros((nq, stride), dtype=torch.float64, device="cuda")
    d_mas = mas if on_dev else torch.zeros((nq, stride), dtype=torch.float64, device="cuda")
    d_sz = sizes if (isinstance(sizes, torch.Tensor) and sizes.is_cuda) else torch.zeros(
        nq, dtype=torch.int64, device="cuda")
    _lib.call("ss_match_pmfs", _lib.ptr(d_sims), nq, nw, _lib.ptr(d_lens), float(theta),
              int(max_len), _lib.ptr(d_sup), _lib.ptr(d_mas), _lib.ptr(d_sz),
              int(d_sup.shape[1]), _lib.stream_ptr())
    if not on_dev:
        w = sup.shape[1]
        sz = d_sz.cpu().numpy()
        hs, hm = d_sup.cpu().numpy(), d_mas.cpu().numpy()
        for q in range(nq):
            k = int(sz[q])
            if k > w:
                raise IndexError(f"output row {q} needs {k} columns, has {w}")
            sup[q, :k] = hs[q, :k]
            mas[q, :k] = hm[q, :k]
        if not isinstance(sizes, torch.Tensor):
            sizes[:] = sz
    elif not (isinstance(sizes, torch.Tensor) and sizes.is_cuda):
        sizes[:] = d_sz.cpu().numpy()


def gittins_min_batch(support: torch.Tensor, masses: torch.Tensor, npts: torch.Tensor,
                      out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched gittins_min on device tensors f64 [n, stride] (warp per law)."""
    n, stride = support.shape
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=support.device)
    _lib.call("ss_gittins_min_batch", _lib.ptr(support), _lib.ptr(masses), _lib.ptr(npts), n,
              stride, _lib.ptr(out), _lib.stream_ptr())
    return out


def gittins_min(support, masses) -> float:
    """min_k (cum_xp + s_k (1 - cum_p)) / cum_p over support points
    (_kernels.py:104-116).  Leading zero mass raises ZeroDivisionError.

    The reference's per-law call: host arrays through ss_gittins_min_host
    (a mapped pinned slot the kernel reads and answers through, no
    allocation); an engine that has many laws uses ``gittins_min_batch``
    (device tensors, one launch)."""
    _lib.require_cuda()
    s = np.ascontiguousarray(support, dtype=np.float64).reshape(-1)
    m = np.ascontiguousarray(masses, dtype=np.float64).reshape(-1)
    if s.size != m.size:
        raise ValueError("support and masses differ in length")
    out = C.c_double()
    # host memory in and out: the library's own per-thread stream and mapped
    # slot (no torch stream lookup, no copy engine, no stream sync)
    _lib.call("ss_gittins_min_host", s.ctypes.data, m.ctypes.data, s.size, C.byref(out), None)
    return out.value


def embed_accumulate_batch(tokens: torch.Tensor, offsets: torch.Tensor, salt: int, dim: int,
                           out: torch.Tensor | None = None) -> torch.Tensor:
    """Feature-hash many prompts at once (warp per prompt) -> f64 [n, dim]."""
    n = offsets.numel() - 1
    if out is None:
        out = torch.empty((n, dim), dtype=torch.float64, device=tokens.device)
    _lib.call("ss_embed_accumulate_batch", _lib.ptr(tokens), _lib.ptr(offsets), n,
              int(salt) & (2**64 - 1), int(dim), _lib.ptr(out), _lib.stream_ptr())
    return out


def embed_accumulate(tokens, salt: int, dim: int) -> np.ndarray:
    """Signed 1-/2-gram feature hash into ``dim`` buckets (_kernels.py:99-102)."""
    _lib.require_cuda()
    t = _dev(np.asarray(tokens, dtype=np.int64).reshape(-1) if not isinstance(tokens, torch.Tensor)
             else tokens.reshape(-1), torch.int64)
    if t.numel() == 0:
        t = torch.zeros(1, dtype=torch.int64, device="cuda")
        offs = torch.tensor([0, 0], dtype=torch.int64, device="cuda")
    else:
        offs = torch.tensor([0, t.numel()], dtype=torch.int64, device="cuda")
    return embed_accumulate_batch(t, offs, salt, dim)[0].cpu().numpy()


def warmup() -> None:
    """Load the library and touch every kernel family once (_kernels.py:167-177)."""
    _lib.load()
    _lib.require_cuda()
    embed_accumulate(np.arange(4, dtype=np.int64), 1, 8)
    gittins_min(np.array([1.0, 2.0]), np.array([0.5, 0.5]))
    sims = np.ones((1, 2), dtype=np.float32)
    lens = np.array([1, 2], dtype=np.int64)
    sup = np.zeros((1, 2))
    mas = np.zeros((1, 2))
    sizes = np.zeros(1, dtype=np.int64)
    match_pmfs(sims, lens, np.float32(0.5), 2, sup, mas, sizes)

"""Seeded synthetic inputs of the BASELINE shapes.

Embeddings: C cluster centroids ~ N(0, I) normalised; each member is
centroid + 0.45 * unit noise, renormalised, then quantised per row to int8
integer vectors round(127 x / max|x|) -- the integer-vector representation
of the reference's feature-hash embeddings (_kernels.py:64-65).  Output
lengths are lognormal per cluster, truncated to [1, max_len].
Input lengths are uniform integers in [1, 4096].

The bank is generated on the device with torch (input preparation only);
queries are generated on the host with numpy, with their fp32 inverse norms
computed by IEEE sqrt/divide exactly as the bank does on device.
"""

from __future__ import annotations

import numpy as np
import torch

__all__ = ["centroids", "make_bank_device", "make_bank_host", "make_queries", "inv_norm_np",
           "inv_norm_device"]


def centroids(n_clusters: int, dim: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((n_clusters, dim)).astype(np.float32)
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    mu = rng.uniform(3.0, 6.5, n_clusters).astype(np.float32)
    return c, mu


def _quantise(x: torch.Tensor) -> torch.Tensor:
    x = x / x.norm(dim=1, keepdim=True)
    return torch.round(127.0 * x / x.abs().amax(dim=1, keepdim=True)).to(torch.int8)


def make_bank_device(n: int, dim: int, n_clusters: int, seed: int, noise: float = 0.45,
                     max_len: int = 2048, chunk: int = 1 << 18, device: str = "cuda",
                     member_seed: int | None = None):
    """(emb int8 [n, dim], lens int32 [n], cluster int64 [n]) on `device`.

    ``seed`` fixes the clusters (centroids and length laws); ``member_seed``
    (default seed + 1) the members, so a trace drawn with another member seed
    shares the bank's clusters."""
    cent, mu = centroids(n_clusters, dim, seed)
    cent_t = torch.as_tensor(cent, device=device)
    mu_t = torch.as_tensor(mu, device=device)
    g = torch.Generator(device=device)
    g.manual_seed(seed + 1 if member_seed is None else member_seed)
    emb = torch.empty((n, dim), dtype=torch.int8, device=device)
    lens = torch.empty(n, dtype=torch.int32, device=device)
    cl_all = torch.empty(n, dtype=torch.int64, device=device)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        cl = torch.randint(0, n_clusters, (m,), generator=g, device=device)
        z = torch.randn((m, dim), generator=g, device=device)
        z = z / z.norm(dim=1, keepdim=True)
        emb[s:s + m] = _quantise(cent_t[cl] + noise * z)
        ln = torch.exp(mu_t[cl] + 0.5 * torch.randn((m,), generator=g, device=device))
        lens[s:s + m] = torch.clamp(torch.round(ln), 1, max_len).to(torch.int32)
        cl_all[s:s + m] = cl
    return emb, lens, cl_all


def make_bank_host(n: int, dim: int, n_clusters: int, seed: int, noise: float = 0.45,
                   max_len: int = 2048, chunk: int = 1 << 17):
    """The same recipe as make_bank_device with numpy on the host (the CPU
    reference arm's bank: same clusters and length laws, numpy's stream of
    members): (emb int8 [n, dim], lens int32 [n])."""
    cent, mu = centroids(n_clusters, dim, seed)
    rng = np.random.default_rng(seed + 1)
    emb = np.empty((n, dim), dtype=np.int8)
    lens = np.empty(n, dtype=np.int32)
    for s in range(0, n, chunk):
        m = min(chunk, n - s)
        cl = rng.integers(0, n_clusters, m)
        z = rng.standard_normal((m, dim), dtype=np.float32)
        z /= np.linalg.norm(z, axis=1, keepdims=True)
        x = cent[cl] + noise * z
        x /= np.linalg.norm(x, axis=1, keepdims=True)
        emb[s:s + m] = np.rint(127.0 * x / np.abs(x).max(axis=1, keepdims=True)).astype(np.int8)
        ln = np.exp(mu[cl] + 0.5 * rng.standard_normal(m, dtype=np.float32))
        lens[s:s + m] = np.clip(np.rint(ln), 1, max_len).astype(np.int32)
    return emb, lens


def inv_norm_np(emb: np.ndarray) -> np.ndarray:
    """fp32 1/sqrt(sum x^2) with IEEE rounding; NaN for a zero row."""
    ss = (emb.astype(np.int64) ** 2).sum(axis=1).astype(np.float32)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.float32(1.0) / np.sqrt(ss)
    r[ss == 0] = np.nan
    return r.astype(np.float32)


def make_queries(nq: int, dim: int, n_clusters: int, seed: int, qseed: int,
                 noise: float = 0.45, max_input: int = 4096):
    """Host (numpy) pending prompts drawn from the same clusters as the bank:
    (q int8 [nq, dim], q_inv f32 [nq], input_len int32 [nq], ids int64 [nq])."""
    cent, _ = centroids(n_clusters, dim, seed)
    rng = np.random.default_rng(qseed)
    cl = rng.integers(0, n_clusters, nq)
    z = rng.standard_normal((nq, dim)).astype(np.float32)
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    x = cent[cl] + noise * z
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = np.rint(127.0 * x / np.abs(x).max(axis=1, keepdims=True)).astype(np.int8)
    I = rng.integers(1, max_input + 1, nq).astype(np.int32)
    ids = np.arange(nq, dtype=np.int64)
    return q, inv_norm_np(q), I, ids


def inv_norm_device(emb: torch.Tensor) -> torch.Tensor:
    """fp32 1/sqrt(sum x^2) on the device (IEEE sqrt and divide, as the bank
    computes it); NaN for a zero row."""
    ss = (emb.to(torch.int32) ** 2).sum(dim=1).to(torch.float32)
    r = 1.0 / torch.sqrt(ss)
    return torch.where(ss == 0, torch.full_like(r, float("nan")), r)

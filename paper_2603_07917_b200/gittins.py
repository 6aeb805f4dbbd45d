"""Gittins index, attained-service conditioning and refresh cadence
(gittins module; index formula PAPER.md:336).

    G(D) = min over support points x_k of E[min(X, x_k)] / P(X <= x_k)

smaller G is served first.  The north-star index
max_a P(S <= a)/E[min(S, a)] is 1/G; ``north_star_index`` returns it.
All arithmetic on laws runs on the GPU: single laws go through the batched
kernels with a batch of one.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .cost import CostModelKind, ResourceBound, cost
from .distribution import DiscreteDistribution, DistributionError

__all__ = ["GittinsConfig", "ServiceProgress", "gittins_index", "gittins_index_batch",
           "condition_on_attained", "refresh_due", "north_star_index", "outlived_index"]


@dataclass(frozen=True)
class GittinsConfig:
    bucket_size_tokens: int = 200
    max_support_points: int = 4096

    def __post_init__(self):
        if self.bucket_size_tokens < 1:
            raise ValueError("bucket_size_tokens must be >= 1")
        if self.max_support_points < 2:
            raise ValueError("max_support_points must be >= 2")


@dataclass(frozen=True)
class ServiceProgress:
    """tokens_generated g, attained cost a = cost(kind, I, g), bucket floor(g/B)."""

    tokens_generated: int
    attained_cost: float
    current_bucket: int

    @classmethod
    def start(cls) -> "ServiceProgress":
        return cls(0, 0.0, 0)

    def advance(self, kind: CostModelKind, input_len: float, g_new: int,
                cfg: GittinsConfig = GittinsConfig()) -> "ServiceProgress":
        return ServiceProgress(int(g_new), cost(kind, input_len, g_new),
                               int(g_new) // cfg.bucket_size_tokens)


def refresh_due(progress: ServiceProgress, g_new: int, cfg: GittinsConfig = GittinsConfig()) -> bool:
    """True iff floor(g_new / bucket) > current bucket."""
    if g_new < progress.tokens_generated:
        raise ValueError("g_new must be >= tokens_generated")
    return (int(g_new) // cfg.bucket_size_tokens) > progress.current_bucket


def outlived_index(kind: CostModelKind, input_len: float, g: int,
                   cfg: GittinsConfig = GittinsConfig()) -> float:
    """One-point law used once a request outlives its whole predicted support
    (SPEC.md:373): bucket_size tokens' worth of further cost."""
    return cost(kind, input_len, g + cfg.bucket_size_tokens) - cost(kind, input_len, g)


def gittins_index_batch(support: torch.Tensor, masses: torch.Tensor, npts: torch.Tensor,
                        attained: torch.Tensor | None = None,
                        outlived: torch.Tensor | None = None,
                        out: torch.Tensor | None = None) -> torch.Tensor:
    """Batched index of conditioned laws on device tensors (warp per law)."""
    n, stride = support.shape
    if out is None:
        out = torch.empty(n, dtype=torch.float64, device=support.device)
    _lib.call("ss_gittins_dist_batch", _lib.ptr(support), _lib.ptr(masses), _lib.ptr(npts),
              _lib.ptr(attained), _lib.ptr(outlived), n, stride, _lib.ptr(out), _lib.stream_ptr())
    return out


def _to_dev(d: DiscreteDistribution):
    s = torch.as_tensor(np.array(d.support, dtype=np.float64), dtype=torch.float64, device="cuda")
    m = torch.as_tensor(np.array(d.masses, dtype=np.float64), dtype=torch.float64, device="cuda")
    return s.reshape(1, -1), m.reshape(1, -1)


def gittins_index(d: DiscreteDistribution) -> float:
    """Gittins index of a cost law."""
    _lib.require_cuda()
    if np.any(np.asarray(d.support) <= 0):
        raise ValueError("Gittins index needs support values > 0 (SPEC.md:330)")
    s, m = _to_dev(d)
    npts = torch.tensor([s.shape[1]], dtype=torch.int64, device="cuda")
    return float(gittins_index_batch(s, m, npts)[0].item())


def north_star_index(d: DiscreteDistribution) -> float:
    """max_a P(S <= a) / E[min(S, a)] = 1 / G."""
    return 1.0 / gittins_index(d)


def condition_on_attained(d: DiscreteDistribution, a: float) -> DiscreteDistribution:
    """Law of (X - a) | X > a: drop points <= a, shift by -a, renormalise
    (SPEC.md:335-343).  P(X > a) = 0 raises DistributionError."""
    _lib.require_cuda()
    if a == 0:
        return d
    s, m = _to_dev(d)
    keep = s[0] > a
    if not bool(keep.any().item()):
        raise DistributionError("already complete under every hypothesis: P(X > a) = 0")
    ss = s[0][keep] - a
    mm = m[0][keep]
    mm = mm / mm.sum()
    return DiscreteDistribution._trusted(ss.cpu().numpy(), mm.cpu().numpy())


def default_kind() -> CostModelKind:
    return ResourceBound()

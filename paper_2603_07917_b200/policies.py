"""Gittins priority and the scheduling total order.

Priority = (primary_key ascending, tie_key = (arrival_time, id)) with smaller
served first.  Only the policies on the north-star path are
provided: ``gittins`` (with bucket refresh) and ``gittins-no-refresh``; the
baseline policies are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .cost import CostModelKind, ResourceBound
from .distribution import DiscreteDistribution
from .gittins import GittinsConfig, ServiceProgress, condition_on_attained, gittins_index, \
    outlived_index
from .scheduler import rank as _rank

__all__ = ["Priority", "priority", "rank_priorities"]


@dataclass(frozen=True, order=True)
class Priority:
    primary_key: float
    tie_key: tuple = (0.0, 0)


def priority(kind: str, request, progress: ServiceProgress, cost_dist: DiscreteDistribution,
             clock: float = 0.0, cost_kind: CostModelKind = ResourceBound(),
             cfg: GittinsConfig = GittinsConfig()) -> Priority:
    """SPEC.md:404-412.  ``gittins``: index of the law conditioned on attained
    cost (refreshed by the caller per refresh_due); ``gittins-no-refresh``:
    index of the admission-time law."""
    if cost_dist is None:
        raise ValueError(f"request {getattr(request, 'id', '?')}: missing prediction")
    tie = (float(getattr(request, "arrival_time", 0.0)), int(getattr(request, "id", 0)))
    if kind == "gittins-no-refresh" or progress.attained_cost == 0:
        return Priority(gittins_index(cost_dist), tie)
    if kind == "gittins":
        if not np.any(cost_dist.support > progress.attained_cost):
            g = outlived_index(cost_kind, request.input_len, progress.tokens_generated, cfg)
            return Priority(g, tie)
        return Priority(gittins_index(condition_on_attained(cost_dist, progress.attained_cost)), tie)
    raise ValueError(f"unsupported policy kind {kind!r} (only gittins policies are on the path)")


def rank_priorities(priorities: list[Priority]) -> np.ndarray:
    """Order of a list of priorities by (primary, arrival, id) via the device
    radix sort.  The tie key is densified to arrival order first (a stable
    host argsort of the tie tuples) so the device sort keys on (G, rank)."""
    n = len(priorities)
    ties = sorted(range(n), key=lambda i: priorities[i].tie_key)
    tie_rank = np.empty(n, dtype=np.int64)
    tie_rank[ties] = np.arange(n)
    G = torch.tensor([p.primary_key for p in priorities], dtype=torch.float64, device="cuda")
    ids = torch.as_tensor(tie_rank, device="cuda")
    return _rank(G, ids).cpu().numpy()

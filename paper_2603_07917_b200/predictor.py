"""Semantic-history output-length predictor (predictor module).

``predict(kind, request, window, fallback)`` keeps the SPEC signature and
returns a DiscreteDistribution of output lengths.  With the north-star top-k,
the neighbour set is top-k by (cos desc, insertion_seq desc) intersected with
cos >= theta; with k >= #matches and bin width 1 it is exactly
the reference's threshold match (_kernels.py:118-138).  Lengths are binned
(width max_len/nbins) and each bin is represented by its conditional mean
length (exact at width 1).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .distribution import DiscreteDistribution
from .history import DEFAULT_SALT, HistoryWindow, embed
from .scheduler import RoundConfig, SageScheduler

__all__ = ["SemanticHistory", "Request", "predict"]


@dataclass(frozen=True)
class SemanticHistory:
    theta: float = 0.8
    min_matches: int = 20
    k: int = 64              # north-star top-k
    max_len: int = 2048
    nbins: int = 2048        # width-1 bins: exact integer lengths

    def __post_init__(self):
        if not 0.0 <= self.theta <= 1.0 and self.theta != -1.0:
            raise ValueError("theta must lie in [0, 1] (or -1 for pure top-k)")
        if self.min_matches < 1:
            raise ValueError("min_matches must be >= 1")


@dataclass
class Request:
    """SPEC.md:25-31 Request (the fields the predictor reads)."""

    id: int
    prompt_tokens: np.ndarray
    input_len: int = 0
    arrival_time: float = 0.0
    embedding: torch.Tensor | None = field(default=None, repr=False)
    inv_norm: torch.Tensor | None = field(default=None, repr=False)

    def __post_init__(self):
        if not self.input_len:
            self.input_len = max(1, len(self.prompt_tokens))


def _embedding(req: Request, dim: int):
    if req.embedding is None:
        req.embedding, req.inv_norm = embed(req.prompt_tokens, DEFAULT_SALT, dim)
    return req.embedding, req.inv_norm


_SCHEDULERS: "weakref.WeakKeyDictionary[HistoryWindow, dict]" = weakref.WeakKeyDictionary()


def _scheduler(window: HistoryWindow, kind: SemanticHistory) -> SageScheduler:
    """One SageScheduler (and its buffers) per (window, predictor config),
    reused across predict calls."""
    per = _SCHEDULERS.setdefault(window, {})
    s = per.get(kind)
    if s is None:
        s = per[kind] = SageScheduler(window, RoundConfig(k=kind.k, theta=kind.theta,
                                                          min_matches=kind.min_matches,
                                                          max_len=kind.max_len, nbins=kind.nbins))
    return s


def predict(kind: SemanticHistory, request: Request, window: HistoryWindow,
            fallback: DiscreteDistribution | None = None) -> DiscreteDistribution:
    """Output-length law of one request.

    Fewer than ``min_matches`` surviving neighbours -> ``fallback`` if given,
    else the empirical law of the whole window; empty window and no fallback
    -> ColdStartError.
    """
    if not isinstance(kind, SemanticHistory):
        raise TypeError(f"unsupported predictor kind: {kind!r}")
    if len(window) == 0:
        if fallback is None:
            raise _lib.ColdStartError("cold start: empty window and no fallback; warm-start the window")
        return fallback
    e, inv = _embedding(request, window.dim)
    sched = _scheduler(window, kind)
    st = sched.predict(e.reshape(1, -1), inv.reshape(1), torch.tensor([request.input_len]))
    if bool(st.used_fb[0].item()) and fallback is not None:
        return fallback
    n = int(st.npts[0].item())
    c = st.pcnt[0, :n].double()
    sv = st.psv[0, :n].double()
    support = (sv / c).cpu().numpy()
    masses = (c / c.sum()).cpu().numpy()
    return DiscreteDistribution._trusted(support, masses)

"""Trace generation and the JSON Lines trace format.

The wire format the c5 replay consumes, restated from the reference's
workload module: ``Request`` records with Poisson arrivals,
clustered prompts (cluster template + fresh noise tokens) and realised
output lengths drawn once from the cluster's truncated length law.

  * ``generate_trace(cfg)``   SPEC.md:48-55 -- pure function of the config
    (numpy ``default_rng(seed)``); i.i.d. exponential gaps of rate lambda;
    cluster chosen with the configured weights; O* truncated to
    [1, O_max] by resampling up to 100 times, then clamping.
  * ``save_trace`` / ``load_trace``  SPEC.md:57-65,82 -- one JSON object per
    line with keys {id, arrival_time, prompt_tokens, input_len,
    true_output_len, cluster_id?}; load re-sorts by (arrival_time, id) with a
    warning when the file is out of order, rejects malformed records with the
    line number (``TraceError``), and an empty file is an empty trace.
  * ``to_replay_trace`` embeds the prompts on the GPU (feature hash ->
    int8 + inverse norm, ``history.embed_batch``) into the device-ready
    ``replay.Trace`` -- ids are the arrival order, as the rank tie-break
    requires.

Host-side plumbing only: this is the input side of the hot path, not the
reference's harness or CLI (out of scope).
"""

from __future__ import annotations

import json
import math
import warnings
from dataclasses import dataclass

import numpy as np

__all__ = ["Request", "LengthLaw", "ClusterSpec", "WorkloadConfig", "TraceError",
           "generate_trace", "save_trace", "load_trace", "to_replay_trace"]


class TraceError(ValueError):
    """A malformed trace record or configuration (names the field / line)."""


@dataclass(frozen=True)
class Request:
    """One inference job."""

    id: int
    arrival_time: float
    prompt_tokens: tuple
    input_len: int
    true_output_len: int
    cluster_id: int | None = None

    def __post_init__(self):
        if self.input_len < 1 or self.true_output_len < 1:
            raise TraceError(f"request {self.id}: input_len and true_output_len must be >= 1")
        if self.input_len != len(self.prompt_tokens):
            raise TraceError(f"request {self.id}: input_len {self.input_len} != prompt length "
                             f"{len(self.prompt_tokens)}")
        if not self.arrival_time >= 0:
            raise TraceError(f"request {self.id}: arrival_time must be >= 0")


@dataclass(frozen=True)
class LengthLaw:
    """Parametric output-length law: lognormal(mu, sigma),
    geometric(p) or bimodal(v1, p1, v2)."""

    kind: str
    params: tuple

    def __post_init__(self):
        k, p = self.kind, self.params
        if k == "lognormal":
            ok = len(p) == 2 and p[1] > 0
        elif k == "geometric":
            ok = len(p) == 1 and 0 < p[0] <= 1
        elif k == "bimodal":
            ok = len(p) == 3 and 0 < p[1] < 1 and p[0] >= 1 and p[2] >= 1
        else:
            raise TraceError(f"length_law: unknown kind {k!r}")
        if not ok:
            raise TraceError(f"length_law: bad parameters {p!r} for {k}")

    def draw(self, rng: np.random.Generator) -> int:
        k, p = self.kind, self.params
        if k == "lognormal":
            return int(round(float(rng.lognormal(p[0], p[1]))))
        if k == "geometric":
            return int(rng.geometric(p[0]))
        return int(p[0] if rng.random() < p[1] else p[2])


@dataclass(frozen=True)
class ClusterSpec:
    """Prompt cluster: shared template + noise_len random
    suffix tokens; output lengths from ``length_law``."""

    template_tokens: tuple
    noise_len: int
    length_law: LengthLaw
    weight: float = 1.0


@dataclass(frozen=True)
class WorkloadConfig:
    """arrival rate lambda (requests/s), n_requests, seed, O_max
    and the per-cluster specs."""

    lam: float
    n_requests: int
    clusters: tuple
    seed: int = 0
    o_max: int = 2048
    vocab: int = 50_000

    def validate(self):
        if not self.lam > 0:
            raise TraceError("lam: must be > 0")
        if self.n_requests < 1:
            raise TraceError("n_requests: must be >= 1")
        if not self.clusters:
            raise TraceError("clusters: at least one ClusterSpec")
        if self.o_max < 1:
            raise TraceError("o_max: must be >= 1")
        for i, c in enumerate(self.clusters):
            if c.noise_len < 0 or len(c.template_tokens) + c.noise_len < 1:
                raise TraceError(f"clusters[{i}]: prompt would be empty")
            if not c.weight > 0:
                raise TraceError(f"clusters[{i}].weight: must be > 0")


def _truncated(law: LengthLaw, rng, o_max: int) -> int:
    # resample up to 100 times, then clamp (keeps determinism)
    v = law.draw(rng)
    for _ in range(100):
        if 1 <= v <= o_max:
            return v
        v = law.draw(rng)
    return min(max(v, 1), o_max)


def generate_trace(cfg: WorkloadConfig) -> list[Request]:
    """Seeded synthetic trace, sorted by arrival time; ids in arrival order."""
    cfg.validate()
    rng = np.random.default_rng(cfg.seed)
    w = np.array([c.weight for c in cfg.clusters], np.float64)
    w /= w.sum()
    gaps = rng.exponential(1.0 / cfg.lam, cfg.n_requests)
    t = np.cumsum(gaps)
    cl = rng.choice(len(cfg.clusters), size=cfg.n_requests, p=w)
    out = []
    for i in range(cfg.n_requests):
        c = cfg.clusters[int(cl[i])]
        noise = rng.integers(0, cfg.vocab, c.noise_len)
        prompt = tuple(int(x) for x in c.template_tokens) + tuple(int(x) for x in noise)
        o = _truncated(c.length_law, rng, cfg.o_max)
        out.append(Request(i, float(t[i]), prompt, len(prompt), o, int(cl[i])))
    return out


_KEYS = ("id", "arrival_time", "prompt_tokens", "input_len", "true_output_len")


def save_trace(reqs, path: str) -> None:
    """JSON Lines, one request per line; arrival_time written with
    repr precision so load(save(t)) == t exactly."""
    with open(path, "w", encoding="utf-8") as f:
        for r in reqs:
            d = {"id": int(r.id), "arrival_time": float(r.arrival_time),
                 "prompt_tokens": [int(x) for x in r.prompt_tokens], "input_len": int(r.input_len),
                 "true_output_len": int(r.true_output_len)}
            if r.cluster_id is not None:
                d["cluster_id"] = int(r.cluster_id)
            f.write(json.dumps(d, separators=(",", ":")) + "\n")


def load_trace(path: str) -> list[Request]:
    """Parse a JSON Lines trace; malformed record -> TraceError naming the
    line; unsorted input is re-sorted (stable, tie-break by id) with a warning."""
    out = []
    with open(path, "r", encoding="utf-8") as f:
        for ln, line in enumerate(f, 1):
            if not line.strip():
                continue
            try:
                d = json.loads(line)
                missing = [k for k in _KEYS if k not in d]
                if missing:
                    raise TraceError(f"missing {missing}")
                at = float(d["arrival_time"])
                if not math.isfinite(at):
                    raise TraceError("arrival_time must be finite")
                r = Request(int(d["id"]), at, tuple(int(x) for x in d["prompt_tokens"]),
                            int(d["input_len"]), int(d["true_output_len"]),
                            None if d.get("cluster_id") is None else int(d["cluster_id"]))
            except (TraceError, ValueError, TypeError, json.JSONDecodeError) as e:
                raise TraceError(f"{path}:{ln}: {e}") from None
            out.append(r)
    if len({r.id for r in out}) != len(out):
        raise TraceError(f"{path}: duplicate request ids")
    key = [(r.arrival_time, r.id) for r in out]
    if any(key[i] > key[i + 1] for i in range(len(key) - 1)):
        warnings.warn(f"{path}: records not sorted by arrival_time; re-sorted", stacklevel=2)
        out.sort(key=lambda r: (r.arrival_time, r.id))
    return out


def to_replay_trace(reqs, dim: int = 384, salt: int | None = None):
    """Embed the prompts on the GPU (int8 feature hash + fp32 inverse norm,
    history.embed_batch) into a ``replay.Trace``; requests must be in arrival
    order with ids 0..n-1 (the rank tie-break)."""
    from .history import DEFAULT_SALT, embed_batch
    from .replay import Trace

    for i, r in enumerate(reqs):
        if r.id != i:
            raise TraceError(f"replay needs ids in arrival order 0..n-1 (request {i} has id {r.id})")
    emb, inv = embed_batch([r.prompt_tokens for r in reqs], DEFAULT_SALT if salt is None else salt,
                           dim)
    return Trace(emb=emb.cpu().numpy(), inv=inv.cpu().numpy(),
                 input_len=np.array([r.input_len for r in reqs], np.int32),
                 true_len=np.array([r.true_output_len for r in reqs], np.int32))

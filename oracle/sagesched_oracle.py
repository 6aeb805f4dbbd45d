"""CPU oracle for the SageSched per-round scheduling hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this file.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import it, and only as the
checker or the timed CPU baseline -- never as the thing measured or shipped.

Parity status: PINNED.
  * The reference code paths that exist (``servesim._kernels.match_pmfs``,
    ``gittins_min``, ``embed_accumulate``; ``servesim.cost``) are pinned by
    golden vectors produced by running the unmodified reference in the build
    container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``),
    and ``tests/test_oracle_golden.py`` checks this restatement against them.
  * The SPEC-only pieces (query_similar, predict, condition_on_attained,
    refresh_due, priority/rank) are restated from ``/root/reference/SPEC.md``
    and pinned by the SPEC's own examples plus the exact
    reduction to ``match_pmfs`` in the limit k >= #matches, bin width 1.

Semantics follow SURVEY.md App. B (the parity contract, written down in
DESIGN.md section 3):

  score      key[q, j] = fl32(fl32(f32(dot_i8(q, w_j)) * inv_w[j]) * inv_q[q])
             (dot is exact: |dot| <= 384*127^2 < 2^24).
  select     top-k by (key desc, insertion_seq desc),
             intersected with {key >= theta} (_kernels.py:126).
  predict    >= min_matches survivors -> their binned lengths, else the
             whole-window fallback.
  histogram  bin b = (len-1) // w, w = max_len // nbins; integer
             count_b, sum_v_b, sum_v2_b.
  cost       conditional-mean ResourceBound cost per bin
             s_b = (sum_v2_b + 2*I*sum_v_b) * 0.5 / count_b
             (== cost.py:97-99 exactly when w == 1).
  gittins    G = min_k (0.5*P_k + s_k*(T-C_k)) / C_k, the integer-count form
             of _kernels.py:110-115; conditioning on attained cost a
              and the outlived one-point rule.
  rank       ascending (G, id).
"""

from __future__ import annotations

import numpy as np

F32 = np.float32
F64 = np.float64

# --------------------------------------------------------------------------
# embedding hash (restates servesim/_kernels.py:37-102)
# --------------------------------------------------------------------------
_PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_C1 = np.uint64(0x2545F4914F6CDD1D)
_C2 = np.uint64(0xD6E8FEB86659FD93)


def _mix(z):
    """splitmix64 finaliser (_kernels.py:45-48)."""
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def embed_accumulate(tokens, salt: int, dim: int) -> np.ndarray:
    """Signed feature hash of 1- and 2-grams (_kernels.py:51-65, :70-102)."""
    t = np.asarray(tokens, dtype=np.int64).astype(np.uint64)
    with np.errstate(over="ignore"):
        uni = _mix(np.uint64(salt) ^ (t * _PHI + _C1))
        if t.size >= 2:
            bi = _mix(uni[:-1] ^ (uni[1:] * _PHI + _C2))
            h = np.concatenate([uni, bi])
        else:
            h = uni
    out = np.zeros(dim, dtype=np.float64)
    if h.size:
        b = (h % np.uint64(dim)).astype(np.int64)
        neg = ((h >> np.uint64(61)) & np.uint64(1)).astype(bool)
        np.add.at(out, b[~neg], 1.0)
        np.add.at(out, b[neg], -1.0)
    return out


# --------------------------------------------------------------------------
# match_pmfs (restates servesim/_kernels.py:118-138, numba variant)
# --------------------------------------------------------------------------
def match_pmfs(sims, lens, theta, max_len, sup, mas, sizes):
    """Threshold match -> exact integer-length pmf, numba semantics.

    mass = c * (1.0 / total)   (_kernels.py:131-135; the numpy twin uses
    c / total, which differs by <= 1 ulp).  len == 0 is counted in total but
    never emitted (_kernels.py:127,132).
    """
    sims = np.asarray(sims, dtype=F32)
    lens = np.asarray(lens, dtype=np.int64)
    theta = F32(theta)
    for q in range(sims.shape[0]):
        hit = sims[q] >= theta
        matched = lens[hit]
        total = matched.size
        k = 0
        if total > 0:
            counts = np.bincount(matched, minlength=max_len + 1)
            inv = 1.0 / float(total)
            vals = np.flatnonzero(counts[1:]) + 1
            k = vals.size
            sup[q, :k] = vals.astype(F64)
            mas[q, :k] = counts[vals].astype(F64) * inv
        sizes[q] = k


# --------------------------------------------------------------------------
# gittins_min (restates servesim/_kernels.py:104-116)
# --------------------------------------------------------------------------
def gittins_min(support, masses) -> float:
    cum_p = 0.0
    cum_xp = 0.0
    best = np.inf
    for s, m in zip(np.asarray(support, F64), np.asarray(masses, F64)):
        cum_p += m
        cum_xp += s * m
        if cum_p == 0.0:
            raise ZeroDivisionError("float division by zero")
        r = (cum_xp + s * (1.0 - cum_p)) / cum_p
        if r < best:
            best = r
    return float(best)


def condition_on_attained(support, masses, a):
    """Law of (X - a) | X > a.  Returns None if P(X>a)=0."""
    support = np.asarray(support, F64)
    masses = np.asarray(masses, F64)
    keep = support > a
    if not np.any(keep):
        return None
    m = masses[keep]
    return support[keep] - a, m / m.sum()


def gittins_dense_grid(support, masses, step_frac=1e-3):
    """Brute-force inf over a dense Delta grid."""
    support = np.asarray(support, F64)
    masses = np.asarray(masses, F64)
    lo, hi = support[0], support[-1]
    step = max((hi - lo) * step_frac, 1e-12)
    grid = np.concatenate([np.arange(lo, hi + step, step), support])
    best = np.inf
    for d in grid:
        p = masses[support <= d].sum()
        if p <= 0:
            continue
        e = np.sum(np.minimum(support, d) * masses)
        best = min(best, e / p)
    return best


# --------------------------------------------------------------------------
# cost model (restates servesim/cost.py:71-118)
# --------------------------------------------------------------------------
def cost_rb(I, O):
    """ResourceBound cost O^2/2 + I*O (cost.py:79-80)."""
    return O * O / 2.0 + I * O


def cost_vector(kind: str, I: float, lengths, w_in=1.0, w_out=2.0):
    lengths = np.asarray(lengths, F64)
    if kind == "resource-bound":
        return lengths * lengths * 0.5 + I * lengths  # cost.py:98-99
    if kind == "output-only":
        return lengths.copy()  # cost.py:100-101
    if kind == "weighted-sum":
        return w_in * I + w_out * lengths  # cost.py:102-103
    raise ValueError(kind)


# --------------------------------------------------------------------------
# history bank: ring slots, scores, selection
# --------------------------------------------------------------------------
def inv_norm(emb_i8) -> np.ndarray:
    """fp32 1/||x|| of integer vectors, IEEE sqrt and divide; NaN for 0."""
    x = np.asarray(emb_i8).astype(np.int64)
    ss = (x * x).sum(axis=1).astype(F32)  # exact below 2^24 (int8 rows), else one rounding
    with np.errstate(divide="ignore", invalid="ignore"):
        r = F32(1.0) / np.sqrt(ss)
    r[ss == 0] = np.nan
    return r.astype(F32)


def ring_rel(slot, head, capacity):
    """Monotone-in-seq rank of a ring slot: (slot - head) mod capacity."""
    return (np.asarray(slot, np.int64) - head) % capacity


def scores(q_i8, q_inv, w_i8, w_inv) -> np.ndarray:
    """key[q, j] = fl32(fl32(f32(dot) * inv_w[j]) * inv_q[q]).

    int8 vectors: the dot product goes through fp32 BLAS, which is exact:
    every partial sum of int8*int8 products is an integer of magnitude
    < 384*127^2 < 2^24.  Wider integer vectors (feature-hash counts of long
    prompts, _kernels.py:82-95): the exact int64 dot, then one correctly
    rounded conversion to f32.
    """
    q, w = np.asarray(q_i8), np.asarray(w_i8)
    if q.dtype == np.int8 and w.dtype == np.int8:
        d = q.astype(F32) @ w.astype(F32).T
    else:
        d = (q.astype(np.int64) @ w.astype(np.int64).T).astype(F32)
    s = d * np.asarray(w_inv, F32)[None, :]
    return (s * np.asarray(q_inv, F32)[:, None]).astype(F32)


def select_topk(keys_row, seq, k, theta):
    """Indices of top-k by (key desc, seq desc), keeping key >= theta.

    NaN keys (empty slots / degenerate rows) never match.
    """
    keys_row = np.asarray(keys_row, F32)
    valid = np.flatnonzero(~np.isnan(keys_row) & (keys_row >= F32(theta)))
    if valid.size == 0:
        return valid
    order = np.lexsort((-np.asarray(seq)[valid], -keys_row[valid].astype(F64)))
    return valid[order[:k]]


def query_similar(keys_row, seq, theta):
    """every record with cos >= theta, desc sim, tie -> larger seq."""
    return select_topk(keys_row, seq, np.iinfo(np.int64).max, theta)


# --------------------------------------------------------------------------
# binned histogram + cost + gittins, exact integer form
# --------------------------------------------------------------------------
def bin_hist(lens, max_len, nbins):
    """Per-bin (count, sum_v, sum_v2) over lengths in [1, max_len]."""
    lens = np.asarray(lens, np.int64)
    if np.any(lens < 1):
        raise ValueError("length < 1")
    lens = np.minimum(lens, max_len)  # lengths are truncated at O_max
    w = max_len // nbins
    b = (lens - 1) // w
    cnt = np.bincount(b, minlength=nbins).astype(np.int64)
    sv = np.bincount(b, weights=lens.astype(F64), minlength=nbins).astype(np.int64)
    sv2 = np.bincount(b, weights=(lens * lens).astype(F64), minlength=nbins).astype(np.int64)
    return cnt, sv, sv2


def hist_to_points(cnt, sv, sv2, I):
    """Sparse points of the cost law: (bin, count, D) with D = sv2 + 2*I*sv."""
    nz = np.flatnonzero(cnt)
    c = cnt[nz].astype(np.int64)
    D = sv2[nz].astype(np.int64) + 2 * int(I) * sv[nz].astype(np.int64)
    return nz.astype(np.int64), c, D


def points_support(c, D):
    """s_b = D_b * 0.5 / c_b (conditional-mean ResourceBound cost)."""
    return (D.astype(F64) * 0.5) / c.astype(F64)


def gittins_points(c, D, I=None, g=0, bucket=200):
    """Integer-count Gittins with attained-service conditioning.

    attained a = cost(I, g) = g^2/2 + I*g, 2a = A2 = g*g + 2*I*g (int64).
    survivors: s_k > a  <=>  D_k > A2 * c_k
    d_k = D_k - A2*c_k, P'_k / C'_k prefix sums over survivors, T' = C'_last:
    ratio_k  = (0.5*P'_k + (d_k/(2 c_k))*(T'-C'_k)) / C'_k      (_kernels.py:113
             = (P'_k*c_k + d_k*(T'-C'_k)) / (2*c_k*C'_k)          with masses c/T')
    evaluated in that second form: exact int64 sums, f64 products, ONE divide.
    none survive -> cost(I, g+bucket) - cost(I, g)
    Same operation order as the CUDA kernels (no FMA), so bit-identical.
    """
    c = np.asarray(c, np.int64)
    D = np.asarray(D, np.int64)
    A2 = 0 if (I is None or g == 0) else int(g) * int(g) + 2 * int(I) * int(g)
    surv = D > A2 * c
    if not np.any(surv):
        gb = g + bucket
        return float((gb * gb - g * g) * 0.5 + float(I) * bucket)
    cs = c[surv]
    Ds = D[surv] - A2 * cs
    C = np.cumsum(cs)
    P = np.cumsum(Ds)
    T = C[-1]
    num = P.astype(F64) * cs.astype(F64) + Ds.astype(F64) * (T - C).astype(F64)
    ratio = num / ((2.0 * cs.astype(F64)) * C.astype(F64))
    return float(ratio.min())


def predict_round(keys, seq, lens, I, k, theta, min_matches, max_len, nbins,
                  window_lens):
    """Stages 1b-3 for a batch of queries given the full key matrix.

    Returns a list of dicts with neighbours, used_fallback, points and G.
    ``window_lens`` = lengths of every valid record (fallback source).
    """
    fb = bin_hist(window_lens, max_len, nbins)
    out = []
    for q in range(keys.shape[0]):
        nbr = select_topk(keys[q], seq, k, theta)
        used_fb = nbr.size < min_matches
        h = fb if used_fb else bin_hist(lens[nbr], max_len, nbins)
        bins, c, D = hist_to_points(*h, I[q])
        G = gittins_points(c, D)
        out.append(dict(nbr=nbr, used_fallback=used_fb, bins=bins, c=c, D=D,
                        G=G, support=points_support(c, D),
                        masses=c.astype(F64) / float(c.sum())))
    return out


def rank(G, ids):
    """Ascending (G, id) total order. Returns a permutation."""
    return np.lexsort((np.asarray(ids), np.asarray(G, F64)))


def pack_batch(perm, I, g, kv_capacity, max_batch, mode="cut"):
    """Engine batch formation, SPEC.md:470 step 3 (pure-Python restatement).

    Walk ``perm`` (ascending priority); request r projects I[r] + g[r] + 1 KV
    tokens (I + 1 when not yet prefilled, g = 0).  "cut": admit while the
    running sum stays <= K and the count <= B, stopping at the first request
    that does not fit.  "skip": a request that does not fit is passed over and
    the scan continues.  Any request with I + 1 > K raises ValueError
    ("request cannot fit", SPEC.md engine errors).  Returns (batch, tokens).
    """
    I = [int(x) for x in I]
    g = [int(x) for x in g]
    for r, i in enumerate(I):
        if i + 1 > kv_capacity:
            raise ValueError(f"request {r} cannot fit: I + 1 = {i + 1} > K = {kv_capacity}")
    batch, used = [], 0
    for r in perm:
        r = int(r)
        if len(batch) >= max_batch:
            break
        t = I[r] + g[r] + 1
        if used + t <= kv_capacity:
            batch.append(r)
            used += t
        elif mode == "cut":
            break
    return batch, used


def refresh_due(g_old, g_new, bucket=200):
    """SPEC.md:345-353."""
    return (g_new // bucket) > (g_old // bucket)


# --------------------------------------------------------------------------
# synthetic inputs shared by tests (seeded)
# --------------------------------------------------------------------------
def make_bank(n, dim, n_clusters, seed, noise=0.45, max_len=2048):
    """Clustered int8 embeddings + per-cluster lengths, for CPU-sized tests."""
    rng = np.random.default_rng(seed)
    cent = rng.standard_normal((n_clusters, dim)).astype(F32)
    cent /= np.linalg.norm(cent, axis=1, keepdims=True)
    cl = rng.integers(0, n_clusters, n)
    x = cent[cl] + noise * _unit(rng, n, dim)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = np.rint(127.0 * x / np.abs(x).max(axis=1, keepdims=True)).astype(np.int8)
    mu = rng.uniform(3.0, 6.5, n_clusters)
    lens = np.clip(np.rint(np.exp(mu[cl] + 0.5 * rng.standard_normal(n))), 1, max_len)
    return q, lens.astype(np.int32), cl, cent


def _unit(rng, n, dim):
    z = rng.standard_normal((n, dim)).astype(F32)
    return z / np.linalg.norm(z, axis=1, keepdims=True)

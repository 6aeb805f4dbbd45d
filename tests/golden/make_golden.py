"""Generate golden vectors by running the UNMODIFIED reference (servesim).

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nbcache PYTHONDONTWRITEBYTECODE=1 \
        PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/reference_golden.npz.  Every array in it was produced by
calling the reference's own public functions:
  servesim._kernels.match_pmfs     (_kernels.py:118-138, numba path)
  servesim._kernels.gittins_min    (_kernels.py:104-116)
  servesim._kernels.embed_accumulate (_kernels.py:99-102)
  servesim.cost.cost / remaining_cost / cost_distribution (cost.py:71-118)
"""

from __future__ import annotations

import os
import sys

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
sys.dont_write_bytecode = True
sys.path.insert(0, os.environ.get("SERVESIM_SRC", "/root/reference/pkg/src"))

from servesim import _kernels as K  # noqa: E402
from servesim import cost as C  # noqa: E402
from servesim.distribution import DiscreteDistribution  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_golden.npz")


def main() -> None:
    assert K.HAVE_NUMBA, "golden vectors must come from the numba path"
    K.warmup()
    rng = np.random.default_rng(20260317)
    g = {}

    # ---- match_pmfs: threshold match -> exact-length pmf -------------------
    nq, nw, max_len = 24, 700, 96
    sims = rng.uniform(-1.0, 1.0, (nq, nw)).astype(np.float32)
    sims[3] = -1.0  # a query with zero matches
    sims[5, ::7] = np.float32(0.5)  # exact-threshold ties (>= must match)
    lens = rng.integers(1, max_len + 1, nw).astype(np.int64)
    lens[::97] = 0  # len 0: counted in total, never emitted (_kernels.py:127,132)
    sup = np.zeros((nq, max_len + 1))
    mas = np.zeros((nq, max_len + 1))
    sizes = np.zeros(nq, dtype=np.int64)
    K.match_pmfs(sims, lens, np.float32(0.5), max_len, sup, mas, sizes)
    g.update(mp_sims=sims, mp_lens=lens, mp_theta=np.float32(0.5), mp_max_len=max_len,
             mp_sup=sup, mp_mas=mas, mp_sizes=sizes)

    # ---- gittins_min on random pmfs (2..300 points, interior zero masses) --
    n = 300
    npts = rng.integers(1, 300, n)
    P = int(npts.max())
    gs = np.zeros((n, P))
    gm = np.zeros((n, P))
    gv = np.zeros(n)
    for i in range(n):
        k = int(npts[i])
        s = np.sort(rng.choice(np.arange(1, 100000), k, replace=False)).astype(np.float64)
        s = s * rng.uniform(0.01, 50.0)
        m = rng.dirichlet(np.full(k, rng.uniform(0.05, 3.0)))
        if k > 3 and i % 5 == 0:
            m[1:k:3] = 0.0  # interior zeros are harmless in the reference
            m = m / m.sum()
        gs[i, :k] = s
        gm[i, :k] = m
        gv[i] = K.gittins_min(s, m)
    g.update(gm_support=gs, gm_masses=gm, gm_npts=npts, gm_value=gv)

    # ---- embed_accumulate ---------------------------------------------------
    toks = []
    offs = [0]
    for i in range(40):
        L = int(rng.integers(0, 300)) if i else 1
        toks.append(rng.integers(0, 200000, L))
        offs.append(offs[-1] + L)
    tok = np.concatenate(toks).astype(np.int64)
    dims = [384, 256, 17]
    emb = {}
    for d in dims:
        emb[d] = np.stack([K.embed_accumulate(tok[offs[i]:offs[i + 1]], 0xC0FFEE, d)
                           for i in range(40)])
    g.update(em_tokens=tok, em_offsets=np.array(offs, np.int64), em_salt=np.uint64(0xC0FFEE),
             em_384=emb[384], em_256=emb[256], em_17=emb[17])

    # ---- cost model ---------------------------------------------------------
    rb, oo, ws = C.ResourceBound(), C.OutputOnly(), C.WeightedSum(1.0, 2.0)
    Is = rng.integers(1, 4097, 200).astype(np.float64)
    Os = rng.integers(0, 2049, 200).astype(np.float64)
    os_ = np.floor(Os * rng.uniform(0, 1, 200))
    g["cost_I"], g["cost_O"], g["cost_o"] = Is, Os, os_
    g["cost_rb"] = np.array([C.cost(rb, i, o) for i, o in zip(Is, Os)])
    g["cost_oo"] = np.array([C.cost(oo, i, o) for i, o in zip(Is, Os)])
    g["cost_ws"] = np.array([C.cost(ws, i, o) for i, o in zip(Is, Os)])
    g["cost_rem"] = np.array([C.remaining_cost(rb, i, o, x) for i, o, x in zip(Is, Os, os_)])
    # cost_distribution on integer-length pmfs
    cd_sup = np.zeros((50, 64))
    cd_out = np.zeros((50, 64))
    cd_mas = np.zeros((50, 64))
    cd_n = np.zeros(50, np.int64)
    cd_I = rng.integers(1, 4097, 50).astype(np.float64)
    for i in range(50):
        k = int(rng.integers(1, 65))
        s = np.sort(rng.choice(np.arange(1, 2049), k, replace=False)).astype(np.float64)
        m = rng.dirichlet(np.ones(k))
        d = DiscreteDistribution(s, m)
        out = C.cost_distribution(rb, cd_I[i], d)
        cd_sup[i, :k], cd_mas[i, :k], cd_out[i, :k], cd_n[i] = d.support, d.masses, out.support, k
    g.update(cd_sup=cd_sup, cd_mas=cd_mas, cd_out=cd_out, cd_n=cd_n, cd_I=cd_I)

    np.savez_compressed(OUT, **g)
    print("wrote", OUT, os.path.getsize(OUT), "bytes")


if __name__ == "__main__":
    main()

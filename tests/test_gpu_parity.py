"""GPU parity: every kernel on the hot path against the CPU oracle (which is
itself pinned to the reference by tests/test_oracle_golden.py) and against
the reference's golden vectors.  Bars (north star): neighbour sets, counts
and orderings bit-exact; Gittins/cost bit-exact here (the integer form is
deterministic), general-law Gittins within 1e-12 relative."""

import numpy as np
import pytest
import torch

from oracle import sagesched_oracle as O

pytestmark = pytest.mark.gpu


def _t(x, dtype=None):
    t = torch.as_tensor(np.ascontiguousarray(x), device="cuda")
    return t.to(dtype) if dtype is not None else t


# ------------------------------------------------------- reference compat --
def test_match_pmfs_bit_exact_vs_reference(cuda, golden):
    from paper_2603_07917_b200 import _kernels as K
    g = golden
    nq = g["mp_sims"].shape[0]
    sup = np.zeros_like(g["mp_sup"])
    mas = np.zeros_like(g["mp_mas"])
    sizes = np.zeros(nq, np.int64)
    K.match_pmfs(g["mp_sims"], g["mp_lens"], g["mp_theta"], int(g["mp_max_len"]), sup, mas, sizes)
    assert np.array_equal(sizes, g["mp_sizes"])
    for q in range(nq):
        k = sizes[q]
        assert np.array_equal(sup[q, :k], g["mp_sup"][q, :k])
        assert np.array_equal(mas[q, :k], g["mp_mas"][q, :k])


def test_match_pmfs_theta_compared_in_f64(cuda, golden):
    """A Python-float theta that is not an f32 value (0.7): numba promotes
    the f32 sim to f64 for the compare, so a sim equal to f32(0.7) (just
    below 0.7) does not match; an np.float32 theta matches it."""
    from paper_2603_07917_b200 import _kernels
    t32 = np.float32(0.7)
    sims = np.array([[t32, np.nextafter(t32, np.float32(2)), np.float32(0.5)]], np.float32)
    lens = np.array([3, 5, 9], np.int64)
    for theta, want in ((0.7, [5]), (t32, [3, 5])):
        sup = np.zeros((1, 16))
        mas = np.zeros((1, 16))
        sz = np.zeros(1, np.int64)
        _kernels.match_pmfs(sims, lens, theta, 16, sup, mas, sz)
        assert list(sup[0, :sz[0]]) == want, theta
        ref = _ref_kernels()
        if ref is not None:
            s2, m2, z2 = np.zeros((1, 16)), np.zeros((1, 16)), np.zeros(1, np.int64)
            ref.match_pmfs(sims, lens, theta, 16, s2, m2, z2)
            assert np.array_equal(s2, sup) and np.array_equal(m2, mas) and np.array_equal(z2, sz)


def _ref_kernels():
    """The unmodified reference module when baseline/_ref is installed (numba)."""
    import os
    import sys
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(ref):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from servesim import _kernels
        return _kernels
    except Exception:
        return None


def test_match_pmfs_out_of_range_len_raises(cuda):
    from paper_2603_07917_b200 import _kernels as K
    sims = np.ones((1, 3), np.float32)
    with pytest.raises(ValueError):
        K.match_pmfs(sims, np.array([1, 2, 99]), np.float32(0.5), 8, np.zeros((1, 9)),
                     np.zeros((1, 9)), np.zeros(1, np.int64))


def test_gittins_min_vs_reference(cuda, golden):
    from paper_2603_07917_b200 import _kernels as K
    g = golden
    out = K.gittins_min_batch(_t(g["gm_support"]), _t(g["gm_masses"]), _t(g["gm_npts"]))
    got = out.cpu().numpy()
    np.testing.assert_allclose(got, g["gm_value"], rtol=1e-12, atol=0)
    assert K.gittins_min(np.array([1.0, 9.0]), np.array([0.5, 0.5])) == 2.0
    for c in (1.0, 5.0, 1000.0):
        assert K.gittins_min(np.array([c]), np.array([1.0])) == c
    with pytest.raises(ZeroDivisionError):
        K.gittins_min(np.array([1.0, 2.0]), np.array([0.0, 1.0]))
    assert K.gittins_min(np.zeros(0), np.zeros(0)) == np.inf


def test_percall_paths_match_batch(cuda):
    """The per-call drop-ins (mapped slot up to 2048 points, staged copies
    above) give bit-identical values to the batched kernels, for every size
    around the warp and slot boundaries, and from several threads at once
    (the slot is per thread)."""
    import threading

    from paper_2603_07917_b200 import _kernels as K
    from paper_2603_07917_b200 import cost as Cst
    from paper_2603_07917_b200.distribution import DiscreteDistribution
    rng = np.random.default_rng(11)
    laws = []
    for n in (1, 2, 31, 32, 33, 64, 511, 512, 2047, 2048, 2049, 5000):
        sup = np.sort(rng.choice(np.arange(1, 10 * n + 10), n, replace=False)).astype(np.float64)
        mas = rng.random(n) + 0.01
        mas /= mas.sum()
        laws.append((sup, mas))
    for sup, mas in laws:
        n = sup.size
        ref = K.gittins_min_batch(_t(sup[None]), _t(mas[None]), _t(np.array([n], np.int64)))
        assert K.gittins_min(sup, mas) == ref.item(), n
        I = float(rng.integers(1, 4000))
        got = Cst.cost_distribution(Cst.ResourceBound(), I, DiscreteDistribution(sup, mas))
        want = Cst.cost_distribution_batch(Cst.ResourceBound(), _t(np.array([I])), _t(sup[None]),
                                           _t(np.array([n], np.int64)))
        np.testing.assert_array_equal(got.support, want[0, :n].cpu().numpy())
    expect = [K.gittins_min(s_, m_) for s_, m_ in laws]
    errs = []

    def worker():
        torch.cuda.set_device(0)
        for _ in range(20):
            for (s_, m_), e in zip(laws, expect):
                if K.gittins_min(s_, m_) != e:
                    errs.append(s_.size)

    th = [threading.Thread(target=worker) for _ in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs


def test_embed_vs_reference(cuda, golden):
    from paper_2603_07917_b200 import _kernels as K
    g = golden
    t, offs = _t(g["em_tokens"]), _t(g["em_offsets"])
    for d in (384, 256, 17):
        got = K.embed_accumulate_batch(t, offs, int(g["em_salt"]), d).cpu().numpy()
        assert np.array_equal(got, g[f"em_{d}"])
    assert np.array_equal(K.embed_accumulate(g["em_tokens"][:5], int(g["em_salt"]), 384),
                          O.embed_accumulate(g["em_tokens"][:5], int(g["em_salt"]), 384))


def test_embed_quantize_and_push(cuda):
    from paper_2603_07917_b200.history import embed_batch, DEFAULT_SALT
    rng = np.random.default_rng(3)
    prompts = [rng.integers(0, 50000, int(rng.integers(1, 200))) for _ in range(50)] + [[]]
    e, inv = embed_batch(prompts, DEFAULT_SALT, 384)
    ref = np.stack([O.embed_accumulate(p, DEFAULT_SALT, 384) for p in prompts]).astype(np.int8)
    assert np.array_equal(e.cpu().numpy(), ref)
    ri = O.inv_norm(ref)
    gi = inv.cpu().numpy()
    assert np.array_equal(np.isnan(gi), np.isnan(ri))
    assert np.array_equal(gi[~np.isnan(ri)], ri[~np.isnan(ri)])


def _long_prompts(rng, n_normal, dim=384):
    """Normal prompts plus long ones that repeat a token 300-600 times (their
    feature-hash buckets leave the int8 range, _kernels.py:82-95)."""
    normal = [rng.integers(0, 50000, int(rng.integers(5, 200))) for _ in range(n_normal)]
    longp = []
    for j in range(6):
        tok = int(rng.integers(0, 50000))
        body = np.concatenate([np.full(300 + 50 * j, tok), rng.integers(0, 50000, 40 + j)])
        longp.append(body)
    return normal, longp


def test_embed_wide_prompt_exact(cuda):
    """A prompt with 300+ repeats of one token: the device embedding keeps the
    exact counts (int16), equal to the reference embed_accumulate, with the
    inverse norm of the exact sum of squares."""
    from paper_2603_07917_b200.history import DEFAULT_SALT, embed_batch
    rng = np.random.default_rng(8)
    normal, longp = _long_prompts(rng, 10)
    prompts = normal + longp
    e, inv = embed_batch(prompts, DEFAULT_SALT, 384)
    assert e.dtype == torch.int16
    ref = np.stack([O.embed_accumulate(p, DEFAULT_SALT, 384) for p in prompts]).astype(np.int64)
    assert np.abs(ref[len(normal):]).max() >= 300
    assert np.array_equal(e.cpu().numpy().astype(np.int64), ref)
    assert np.array_equal(inv.cpu().numpy(), O.inv_norm(ref))
    e8, _ = embed_batch(normal, DEFAULT_SALT, 384)  # no wide row: the int8 layout
    assert e8.dtype == torch.int8 and np.array_equal(e8.cpu().numpy(), ref[:len(normal)])


@pytest.mark.parametrize("theta", [0.3, -1.0])
def test_wide_rows_and_queries_bit_exact(cuda, theta):
    """embed -> push -> top-k / round with long prompts on both sides: wide
    rows in the bank (among int8 rows), wide queries in the batch (among int8
    queries), near-duplicates of the wide prompts so that wide rows are the
    true neighbours; neighbour lists and Gittins indices equal the oracle's
    bit for bit (the TS kernel at nq > 128, the streaming kernel below)."""
    from paper_2603_07917_b200.history import DEFAULT_SALT, HistoryWindow, embed_batch
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    rng = np.random.default_rng(12)
    n = 5000
    bank_e, bank_l, _, _ = O.make_bank(n, 384, 40, 2)
    normal, longp = _long_prompts(rng, 4)
    le, _ = embed_batch(longp, DEFAULT_SALT, 384)
    le = le.cpu().numpy()
    # bank: int8 rows, then the long prompts and perturbed copies of them
    wide_rows = np.concatenate([le, le + rng.integers(-3, 4, le.shape), le * 2]).astype(np.int16)
    rows = np.concatenate([bank_e.astype(np.int16), wide_rows])
    lens = np.concatenate([bank_l, rng.integers(1, 2049, wide_rows.shape[0]).astype(np.int32)])
    w = HistoryWindow(rows.shape[0] + 64, 384)
    w.push(bank_e[:2500], bank_l[:2500])              # int8 push
    w.push(rows[2500:], lens[2500:])                  # int16 push: int8 rows + wide rows
    seq = np.arange(rows.shape[0])
    rinv = O.inv_norm(rows)
    for nq in (40, 300):
        q8 = O.make_bank(nq, 384, 40, 2 + nq)[0].astype(np.int16)
        q = np.concatenate([le.astype(np.int16), (le[:3] + 1).astype(np.int16), q8])[:nq]
        qi = O.inv_norm(q)
        keys = O.scores(q, qi, rows, rinv)
        comp, ln = w.topk(q, qi, 32, theta)
        key, gseq, _ = w.decode(comp)
        key, gseq, ln = key.cpu().numpy(), gseq.cpu().numpy(), ln.cpu().numpy()
        for i in range(nq):
            sel = O.select_topk(keys[i], seq, 32, theta)
            m = sel.size
            assert np.array_equal(gseq[i, :m], seq[sel]), (nq, i)
            assert np.array_equal(key[i, :m], keys[i, sel]), (nq, i)
            assert np.array_equal(ln[i, :m], lens[sel]), (nq, i)
        # the wide rows are found: the first query's best neighbour is its own prompt
        assert gseq[0, 0] >= n
        I = rng.integers(1, 4097, nq).astype(np.int32)
        ids = np.arange(nq, dtype=np.int64)
        cfg = RoundConfig(k=32, theta=theta, min_matches=10, max_len=2048, nbins=64)
        perm, G, _ = SageScheduler(w, cfg).schedule_round(_t(q), _t(qi), _t(I), _t(ids))
        ref = O.predict_round(keys, seq, lens, I, 32, theta, 10, 2048, 64, window_lens=lens)
        Gr = np.array([r["G"] for r in ref])
        assert np.array_equal(G.cpu().numpy(), Gr)
        assert np.array_equal(perm.cpu().numpy(), O.rank(Gr, ids))
    # an int8 push over a wide slot clears it (the ring wraps onto the wide rows)
    w2 = HistoryWindow(8, 384)
    w2.push(wide_rows[:4], np.arange(1, 5, dtype=np.int32))
    w2.push(bank_e[:8], bank_l[:8])  # evicts every wide row
    qq = wide_rows[:1]
    c2, _ = w2.topk(qq, O.inv_norm(qq), 8, -1.0)
    _, s2, _ = w2.decode(c2)
    assert sorted(s2[0].cpu().numpy().tolist()) == list(range(4, 12))


@pytest.mark.parametrize("theta", [0.8, 0.0, -1.0])
def test_query_similar_returns_every_match(cuda, theta):
    """query_similar returns ALL records with cos >=
    theta (theta = -1: the whole window) ordered by cos desc, ties by the
    larger insertion_seq -- beyond any top-k cap -- on a wrapped ring with
    exact duplicates and a wide row."""
    from paper_2603_07917_b200.history import HistoryWindow, query_similar
    n, cap = 12_000, 10_000
    emb, lens, _, _ = O.make_bank(n + 1, 384, 20, 4)
    emb[3000:3030] = emb[n]  # 30 exact duplicates of the query (ties), inside the live window
    rows = emb[:n].astype(np.int16)
    rows[5000] = rows[5000] * 3  # a wide row (|x| up to 381)
    w = HistoryWindow(cap, 384)
    w.push(rows, lens[:n])
    live = np.arange(n - cap, n)
    q = emb[n]
    keys = O.scores(q[None], O.inv_norm(q[None]), rows[live], O.inv_norm(rows[live]))[0]
    seq, cos, ln = query_similar(w, q, O.inv_norm(q[None])[0], theta)
    ref = O.query_similar(keys, live, theta)
    assert seq.size == ref.size and (theta > -1.0 or seq.size == cap)
    assert ref.size > 256 or theta > 0.5
    assert np.array_equal(seq, live[ref]) and np.array_equal(cos, keys[ref])
    assert np.array_equal(ln, lens[live[ref]])


def test_cost_distribution_vs_reference(cuda, golden):
    from paper_2603_07917_b200.cost import ResourceBound, cost_distribution
    from paper_2603_07917_b200.distribution import DiscreteDistribution
    g = golden
    for i in range(g["cd_n"].size):
        k = int(g["cd_n"][i])
        d = DiscreteDistribution(g["cd_sup"][i, :k], g["cd_mas"][i, :k])
        out = cost_distribution(ResourceBound(), g["cd_I"][i], d)
        assert np.array_equal(out.support, g["cd_out"][i, :k])
    # SPEC.md:281
    out = cost_distribution(ResourceBound(), 100, DiscreteDistribution([100, 300], [.5, .5]))
    assert list(out.support) == [15000.0, 75000.0]


def test_gittins_conditioning_spec_examples(cuda):
    from paper_2603_07917_b200.distribution import DiscreteDistribution as DD
    from paper_2603_07917_b200.gittins import condition_on_attained, gittins_index
    d = DD([1.0, 9.0], [0.5, 0.5])
    assert gittins_index(d) == 2.0
    c = condition_on_attained(d, 1.0)
    assert list(c.support) == [8.0] and gittins_index(c) == 8.0
    c = condition_on_attained(DD([2.0, 4.0, 8.0], [0.25, 0.25, 0.5]), 3.0)
    np.testing.assert_allclose(c.support, [1.0, 5.0])
    np.testing.assert_allclose(c.masses, [1 / 3, 2 / 3])


# -------------------------------------------------------------- the bank ---
def test_ring_push_evicts_oldest(cuda):
    from paper_2603_07917_b200.history import HistoryWindow
    rng = np.random.default_rng(0)
    cap, dim = 100, 128
    w = HistoryWindow(cap, dim)
    e = rng.integers(-127, 128, (250, dim)).astype(np.int8)
    L = rng.integers(1, 2049, 250).astype(np.int32)
    w.push(e[:30], L[:30])
    w.push(e[30:], L[30:])  # wraps twice
    assert w.head == 250 and len(w) == cap
    emb, inv, lens, seq = w.tensors()
    seq = seq.cpu().numpy()
    for slot in range(cap):
        s = 150 + ((slot - 150) % cap)  # the newest seq congruent to slot
        assert seq[slot] == s
        assert np.array_equal(emb[slot].cpu().numpy(), e[s])
        assert lens[slot].item() == L[s]
    assert np.array_equal(inv.cpu().numpy(), O.inv_norm(e[seq]))
    with pytest.raises(ValueError):
        w.push(e[:1], np.array([0], np.int32))  # length < 1 rejected


# ------------------------------------------------------- top-k (stage 1) ---
def _bank(n, dim, ncl, seed, nq, cap=None):
    from paper_2603_07917_b200.history import HistoryWindow
    emb, lens, cl, _ = O.make_bank(n + nq, dim, ncl, seed)
    w = HistoryWindow(cap or n, dim)
    w.push(emb[:n], lens[:n])
    q = emb[n:]
    return w, emb[:n], lens[:n], q, O.inv_norm(q)


def _oracle_topk(w, bank_e, q, q_inv, k, theta):
    head, cap = w.head, w.global_capacity
    n = bank_e.shape[0]
    seq = np.arange(n, dtype=np.int64) + max(0, head - n)
    keys = O.scores(q, q_inv, bank_e, O.inv_norm(bank_e))
    return keys, seq, [O.select_topk(keys[i], seq, k, theta) for i in range(q.shape[0])]


def _check_topk(w, comp, keys, seq, ref, k):
    key, gseq, _ = w.decode(comp)
    key, gseq = key.cpu().numpy(), gseq.cpu().numpy()
    for i, sel in enumerate(ref):
        m = sel.size
        assert np.array_equal(gseq[i, :m], seq[sel]), i
        assert np.array_equal(key[i, :m], keys[i, sel]), i
        assert np.all(gseq[i, m:] == -1)


@pytest.mark.parametrize("algo", ["scan", "tcgen05"])
@pytest.mark.parametrize("theta,k", [(0.8, 32), (-1.0, 32), (0.5, 64), (-1.0, 256)])
def test_topk_c1_bit_exact(cuda, algo, theta, k):
    from paper_2603_07917_b200 import _lib
    w, be, bl, q, qi = _bank(10_000, 384, 100, 7, 64)
    keys, seq, ref = _oracle_topk(w, be, q, qi, k, theta)
    if algo == "tcgen05" and k > 64:  # the tcgen05 heaps hold k <= 64: refused, not truncated
        with pytest.raises(NotImplementedError):
            w.topk(q, qi, k, theta, algo)
        return
    comp, ln = w.topk(q, qi, k, theta, algo)
    _check_topk(w, comp, keys, seq, ref, k)
    lens = ln.cpu().numpy()
    for i, sel in enumerate(ref):
        assert np.array_equal(lens[i, :sel.size], bl[sel])


@pytest.mark.parametrize("algo", ["scan", "tcgen05"])
@pytest.mark.parametrize("theta", [-1.0, 0.8])
def test_topk_multi_tile_ring_wrap(cuda, algo, theta):
    """200k-row bank pushed through a wrapping ring (head > capacity), ragged
    nq=300: many 256-row tiles per CTA, stage-ring and TMEM double-buffer wrap."""
    from paper_2603_07917_b200.history import HistoryWindow
    n, cap, dim, nq, k = 260_000, 200_000, 384, 300, 64
    emb, lens, _, _ = O.make_bank(n + nq, dim, 500, 21)
    w = HistoryWindow(cap, dim)
    w.push(emb[:n], lens[:n])  # wraps: slots hold seqs 60000..259999
    q = emb[n:]
    qi = O.inv_norm(q)
    seqs = np.arange(n - cap, n)
    bank_e = emb[n - cap:n]
    keys = O.scores(q, qi, bank_e, O.inv_norm(bank_e))
    ref = [O.select_topk(keys[i], seqs, k, theta) for i in range(nq)]
    comp, ln = w.topk(q, qi, k, theta, algo)
    key, gseq, _ = w.decode(comp)
    key, gseq, ln = key.cpu().numpy(), gseq.cpu().numpy(), ln.cpu().numpy()
    for i, sel in enumerate(ref):
        m = sel.size
        assert np.array_equal(gseq[i, :m], seqs[sel]), i
        assert np.array_equal(key[i, :m], keys[i, sel]), i
        assert np.array_equal(ln[i, :m], lens[seqs[sel]]), i


@pytest.mark.parametrize("theta", [0.8, -1.0])
def test_topk_after_small_pushes(cuda, theta):
    """The bank's per-16-row filter bounds (rewritten after every write) stay
    exact when pushes of odd sizes rewrite parts of 16-row groups and the
    ring wraps several times: TS-kernel top-k equals the oracle's."""
    from paper_2603_07917_b200.history import HistoryWindow
    cap, dim, nq, k = 20_000, 384, 200, 32
    n = 3 * cap + 777
    emb, lens, _, _ = O.make_bank(n + nq, dim, 60, 8)
    w = HistoryWindow(cap, dim)
    rng = np.random.default_rng(4)
    pos = 0
    while pos < n:
        m = int(min(n - pos, rng.integers(1, 700)))
        w.push(emb[pos:pos + m], lens[pos:pos + m])
        pos += m
    q = emb[n:]
    qi = O.inv_norm(q)
    seqs = np.arange(n - cap, n)
    bank_e = emb[n - cap:n]
    keys = O.scores(q, qi, bank_e, O.inv_norm(bank_e))
    ref = [O.select_topk(keys[i], seqs, k, theta) for i in range(nq)]
    comp, ln = w.topk(q, qi, k, theta, "tcgen05")
    key, gseq, _ = w.decode(comp)
    key, gseq = key.cpu().numpy(), gseq.cpu().numpy()
    for i, sel in enumerate(ref):
        m = sel.size
        assert np.array_equal(gseq[i, :m], seqs[sel]), i
        assert np.array_equal(key[i, :m], keys[i, sel]), i


@pytest.mark.parametrize("theta", [0.8, 0.3, 0.0, -1.0])
def test_topk_large_batch_tcgen05(cuda, theta):
    """nq = 1024 (the A-in-TMEM kernel with its integer pre-filter for
    thr > 0), 40k-row bank over 64 clusters: many neighbours per query, so
    heaps fill and the running threshold rises above theta."""
    w, be, bl, q, qi = _bank(40_000, 384, 64, 5, 1024)
    keys, seq, ref = _oracle_topk(w, be, q, qi, 64, theta)
    comp, ln = w.topk(q, qi, 64, theta, "tcgen05")
    _check_topk(w, comp, keys, seq, ref, 64)


@pytest.mark.parametrize("theta", [-1.0, 0.0])
def test_topk_pure_large_bank_bit_exact(cuda, theta):
    """theta <= 0 (the TS kernel's shared slice bounds) on a 300k-row bank
    with 256 queries: every query's top-k equals the oracle's."""
    w, be, bl, q, qi = _bank(300_000, 384, 64, 21, 256)
    keys, seq, ref = _oracle_topk(w, be, q, qi, 64, theta)
    comp, ln = w.topk(q, qi, 64, theta, "tcgen05")
    _check_topk(w, comp, keys, seq, ref, 64)


@pytest.mark.parametrize("layout", ["ts_mixed", "tc_mixed", "tc_resolved"])
@pytest.mark.parametrize("theta", [-1.0, 0.0])
def test_topk_pure_cascade_mixed_tiles(cuda, theta, layout):
    """Pure top-k runs as a cascade (a threshold pass, then the pure top-k
    pass only for query tiles with a query holding fewer than k keys >= the
    threshold), in both the A-in-TMEM kernel and the streaming kernel.  Queries from tight clusters (hundreds of rows >= 0.8) and
    random queries (none) are interleaved so that every query tile mixes
    resolved and unresolved queries, and one tile holds only cluster queries;
    every top-k equals the oracle's."""
    from paper_2603_07917_b200.history import HistoryWindow
    rng = np.random.default_rng(5)
    dim, ncl, per = 384, 8, 300
    cent = rng.standard_normal((ncl, dim)).astype(np.float32)
    cent /= np.linalg.norm(cent, axis=1, keepdims=True)

    def quant(x):
        x = x / np.linalg.norm(x, axis=1, keepdims=True)
        return np.rint(127.0 * x / np.abs(x).max(axis=1, keepdims=True)).astype(np.int8)

    def members(c, n):
        z = rng.standard_normal((n, dim)).astype(np.float32)
        z /= np.linalg.norm(z, axis=1, keepdims=True)
        return quant(cent[c] + 0.2 * z)

    bank = np.concatenate([members(c, per) for c in range(ncl)]
                          + [quant(rng.standard_normal((30_000, dim)).astype(np.float32))])
    bank = bank[rng.permutation(bank.shape[0])]
    lens = rng.integers(1, 2000, bank.shape[0]).astype(np.int32)
    w = HistoryWindow(bank.shape[0], dim)
    w.push(bank, lens)
    qc = np.concatenate([members(c % ncl, 1) for c in range(256)])          # resolved
    qr = quant(rng.standard_normal((128, dim)).astype(np.float32))           # unresolved
    mixed = np.empty((256, dim), np.int8)
    mixed[0::2], mixed[1::2] = qc[:128], qr
    if layout == "ts_mixed":    # 3 query tiles (A-in-TMEM kernel): 0-1 mixed, 2 all resolved
        q = np.concatenate([mixed, qc[128:]])
    elif layout == "tc_mixed":  # one tile (streaming kernel), mixed
        q = mixed[:96]
    else:                       # one tile, every query resolved by the threshold pass
        q = qc[:64]
    qi = O.inv_norm(q)
    keys, seq, ref = _oracle_topk(w, bank, q, qi, 64, theta)
    comp, ln = w.topk(q, qi, 64, theta, "tcgen05")
    _check_topk(w, comp, keys, seq, ref, 64)


@pytest.mark.parametrize("algo", ["scan", "tcgen05"])
def test_topk_edges(cuda, algo):
    """ragged nq (1 and 3: the streaming tcgen05 kernel; 129: the A-in-TMEM
    kernel with a one-query second tile), partially filled ring, exact
    duplicates (ties broken by the larger insertion_seq), a
    degenerate zero query, theta = 0.9, k > rows.  Only k > 64 leaves the
    tcgen05 kernels (their heap capacity); everything else must run there."""
    from paper_2603_07917_b200.history import HistoryWindow
    rng = np.random.default_rng(11)
    dim = 384
    base = rng.integers(-20, 21, (300, dim)).astype(np.int8)
    base[100:110] = base[5]  # exact duplicates -> score ties broken by larger seq
    L = rng.integers(1, 2049, 300).astype(np.int32)
    w = HistoryWindow(1000, dim)  # 700 empty slots
    w.push(base, L)
    ran = 0
    for nq in (1, 3, 129):
        q = rng.integers(-20, 21, (nq, dim)).astype(np.int8)
        q[0] = base[5]
        if nq > 1:
            q[1] = 0  # degenerate (zero) query: no neighbours
        if nq > 2:
            q[2] = base[100]  # a duplicate of the query above: the same 11-way tie
        qi = O.inv_norm(q)
        for k, theta in ((16, -1.0), (64, -1.0), (256, -1.0), (8, 0.9), (64, 0.9), (32, 0.0)):
            if algo == "tcgen05" and k > 64:
                with pytest.raises(NotImplementedError):
                    w.topk(q, qi, k, theta, algo)
                continue
            comp, _ = w.topk(q, qi, k, theta, algo)
            keys = O.scores(q, qi, base, O.inv_norm(base))
            seq = np.arange(300)
            ref = [O.select_topk(keys[i], seq, k, theta) for i in range(nq)]
            _check_topk(w, comp, keys, seq, ref, k)
            # the tie: the 11 identical rows come newest first
            key0, gseq0, _ = w.decode(comp[:1])
            assert gseq0[0, 0].item() == 109 and key0[0, 0].item() == pytest.approx(1.0, abs=1e-6)
            if nq > 1:
                assert int((comp[1] != 0).sum()) == 0
            ran += 1
    assert ran == 3 * (5 if algo == "tcgen05" else 6)


def _oracle_topk_chunked(q, qi, bank_emb_dev, bank_lens, k, theta, chunk=1 << 20):
    """Exact oracle top-k of a few queries against a bank too large to score
    whole on the host: per chunk, the rows at or above the chunk's k-th key
    (ties included) go to a candidate pool, whose select_topk is the global
    one (the pool holds every row of the global top-k)."""
    n = bank_emb_dev.shape[0]
    pool_k = [[] for _ in range(q.shape[0])]
    pool_s = [[] for _ in range(q.shape[0])]
    for s in range(0, n, chunk):
        e = bank_emb_dev[s:s + chunk].cpu().numpy()
        keys = O.scores(q, qi, e, O.inv_norm(e))
        for i in range(q.shape[0]):
            row = keys[i]
            ok = np.flatnonzero(row >= np.float32(theta)) if theta > -1.0 else np.arange(row.size)
            if ok.size > k:
                kth = np.partition(-row[ok], k - 1)[k - 1]
                ok = ok[-row[ok] <= kth]
            pool_k[i].append(row[ok])
            pool_s[i].append(ok + s)
    out = []
    for i in range(q.shape[0]):
        kv, sv = np.concatenate(pool_k[i]), np.concatenate(pool_s[i])
        sel = O.select_topk(kv, sv, k, theta)
        out.append((sv[sel], kv[sel]))
    return out


@pytest.mark.parametrize("theta", [0.8, -1.0])
def test_round_c4_shape_sampled(cuda, theta):
    """BASELINE configs[3] on one GPU: a 16M-row bank and an 8192-request
    round (64 query tiles, a multi-wave grid of the A-in-TMEM kernel).  For
    32 sampled requests the neighbour lists (insertion_seq and key) and the
    Gittins indices equal the oracle's bit for bit; the permutation orders
    every request by (G, id)."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries
    n, dim, nq, k, nbins = 1 << 24, 384, 8192, 64, 128
    emb, lens, _ = make_bank_device(n, dim, 4096, 0)
    w = HistoryWindow(n, dim)
    w.push(emb, lens)
    bl = lens.cpu().numpy()
    del lens
    q, qi, I, ids = make_queries(nq, dim, 4096, 0, qseed=4000)
    cfg = RoundConfig(k=k, theta=theta, min_matches=20, max_len=2048, nbins=nbins)
    perm, G, _ = SageScheduler(w, cfg).schedule_round(_t(q), _t(qi), _t(I), _t(ids))
    G, perm = G.cpu().numpy(), perm.cpu().numpy()
    assert np.array_equal(perm, O.rank(G, ids))
    comp, ln = w.topk(q, qi, k, theta)
    key, gseq, _ = w.decode(comp)
    key, gseq, ln = key.cpu().numpy(), gseq.cpu().numpy(), ln.cpu().numpy()
    smp = np.sort(np.random.default_rng(5).choice(nq, 32, replace=False))
    ref = _oracle_topk_chunked(q[smp], qi[smp], emb, bl, k, theta)
    del emb
    fb = O.bin_hist(bl, 2048, nbins)
    n_topk = 0
    for j, i in enumerate(smp):
        rs, rk = ref[j]
        m = rs.size
        assert np.array_equal(gseq[i, :m], rs) and np.array_equal(key[i, :m], rk), i
        assert np.all(gseq[i, m:] == -1)
        assert np.array_equal(ln[i, :m], bl[rs]), i
        used_fb = m < 20
        h = fb if used_fb else O.bin_hist(bl[rs], 2048, nbins)
        _, c, D = O.hist_to_points(*h, I[i])
        assert G[i] == O.gittins_points(c, D), i
        n_topk += not used_fb
    assert n_topk >= 16  # the top-k path, not only the fallback


# ------------------------------------------------- full round (stages 1-4) --
@pytest.mark.parametrize("algo", ["scan", "tcgen05"])
@pytest.mark.parametrize("nbins,theta", [(64, 0.8), (2048, 0.8), (128, -1.0)])
def test_round_c1_bit_exact(cuda, algo, nbins, theta):
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    w, be, bl, q, qi = _bank(10_000, 384, 100, 7, 64)
    rng = np.random.default_rng(2)
    I = rng.integers(1, 4097, 64).astype(np.int32)
    ids = np.arange(64, dtype=np.int64)
    k = 32
    cfg = RoundConfig(k=k, theta=theta, min_matches=20, max_len=2048, nbins=nbins, algo=algo)
    s = SageScheduler(w, cfg)
    perm, G, out = s.schedule_round(_t(q), _t(qi), _t(I), _t(ids))
    keys, seq, _ = _oracle_topk(w, be, q, qi, k, theta)
    ref = O.predict_round(keys, seq, bl, I, k, theta, 20, 2048, nbins, window_lens=bl)
    Gr = np.array([r["G"] for r in ref])
    assert np.array_equal(G.cpu().numpy(), Gr)
    assert np.array_equal(perm.cpu().numpy(), O.rank(Gr, ids))
    npts = out["npts"].cpu().numpy()
    for i, r in enumerate(ref):
        assert npts[i] == r["c"].size
        assert np.array_equal(out["pcnt"][i, :npts[i]].cpu().numpy(), r["c"])
        assert np.array_equal(out["pD"][i, :npts[i]].cpu().numpy(), r["D"])
        assert np.array_equal(out["pbin"][i, :npts[i]].cpu().numpy(), r["bins"])
        assert bool(out["used_fb"][i].item()) == r["used_fallback"]
    # host (plugin) entry point gives the same answer
    ph, Gh = s.schedule_round_host(q, qi, I, ids)
    assert np.array_equal(Gh, Gr) and np.array_equal(ph, O.rank(Gr, ids))


@pytest.mark.parametrize("theta", [0.8, -1.0])
def test_round_c2_full_size_sampled(cuda, theta):
    """BASELINE configs[1] at full size (1M-row bank, 1024 requests, k = 64,
    128 bins, the bench's synthetic data; theta = -1 is the pure top-k kernel
    with cross-slice bound sharing): Gittins indices of 32 sampled
    requests equal the oracle's bit for bit (the oracle scores those requests
    against the whole bank), and the permutation orders every request by
    (G, id)."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries
    n, dim, nq, k, nbins = 1 << 20, 384, 1024, 64, 128
    emb, lens, _ = make_bank_device(n, dim, 4096, 0)
    w = HistoryWindow(n, dim)
    w.push(emb, lens)
    q, qi, I, ids = make_queries(nq, dim, 4096, 0, qseed=1000)
    cfg = RoundConfig(k=k, theta=theta, min_matches=20, max_len=2048, nbins=nbins)
    perm, G, _ = SageScheduler(w, cfg).schedule_round(_t(q), _t(qi), _t(I), _t(ids))
    G, perm = G.cpu().numpy(), perm.cpu().numpy()
    assert np.array_equal(perm, O.rank(G, ids))
    be, bl = emb.cpu().numpy(), lens.cpu().numpy()
    del emb, lens
    binv = O.inv_norm(be)
    smp = np.random.default_rng(3).choice(nq, 32, replace=False)
    keys = np.concatenate([O.scores(q[smp], qi[smp], be[s:s + (1 << 18)], binv[s:s + (1 << 18)])
                           for s in range(0, n, 1 << 18)], axis=1)
    ref = O.predict_round(keys, np.arange(n), bl, I[smp], k, theta, 20, 2048, nbins, window_lens=bl)
    assert np.array_equal(G[smp], np.array([r["G"] for r in ref]))
    assert sum(not r["used_fallback"] for r in ref) >= 16  # the top-k path, not only the fallback


def test_round_host_graph_replay(cuda):
    """The plugin call with pinned host buffers: calls 1-2 run eagerly, the
    repeat is captured and later calls replay one graph (H2D + round + D2H).
    New buffer contents and a bank push (head moves) must be honoured."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    n, nq, k, nbins = 10_000, 300, 32, 64
    emb, lens, _, _ = O.make_bank(n + 500 + 2 * nq, 384, 100, 13)
    w = HistoryWindow(12_000, 384)
    w.push(emb[:n], lens[:n])
    qa, qb = emb[n + 500:n + 500 + nq], emb[n + 500 + nq:]
    rng = np.random.default_rng(4)
    I = rng.integers(1, 4097, nq).astype(np.int32)
    ids = np.arange(nq, dtype=np.int64)
    s = SageScheduler(w, RoundConfig(k=k, theta=0.8, min_matches=20, max_len=2048, nbins=nbins))

    def pin(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    hq, hqi, hI, hids = pin(qa), pin(O.inv_norm(qa)), pin(I), pin(ids)
    G = torch.empty(nq, dtype=torch.float64).pin_memory().numpy()
    perm = torch.empty(nq, dtype=torch.int64).pin_memory().numpy()

    def expect(q, nb):
        be, bl = emb[:nb], lens[:nb]
        keys = O.scores(q, O.inv_norm(q), be, O.inv_norm(be))
        ref = O.predict_round(keys, np.arange(nb), bl, I, k, 0.8, 20, 2048, nbins, window_lens=bl)
        Gr = np.array([r["G"] for r in ref])
        return Gr, O.rank(Gr, ids)

    Ga, pa = expect(qa, n)
    Gb, pb = expect(qb, n)
    for it in range(5):
        q = qb if it == 3 else qa
        hq[:] = q
        hqi[:] = O.inv_norm(q)
        s.schedule_round_host(hq, hqi, hI, hids, G, perm)
        Gr, pr = (Gb, pb) if it == 3 else (Ga, pa)
        assert np.array_equal(G, Gr) and np.array_equal(perm, pr), it
    w.push(emb[n:n + 500], lens[n:n + 500])
    Gc, pc = expect(qa, n + 500)
    for it in range(3):
        s.schedule_round_host(hq, hqi, hI, hids, G, perm)
        assert np.array_equal(G, Gc) and np.array_equal(perm, pc), it


def test_round_host_input_paths(cuda):
    """The host-buffer call reads pinned inputs with one gather kernel and
    pageable ones with copies: both, with and without ids, and pinned views
    that are not 16-byte aligned (ragged nq), give the same G and order."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    n, nq = 8_000, 301
    emb, lens, _, _ = O.make_bank(n + nq, 384, 100, 21)
    w = HistoryWindow(n, 384)
    w.push(emb[:n], lens[:n])
    q = emb[n:]
    qi = O.inv_norm(q)
    I = np.random.default_rng(5).integers(1, 4097, nq).astype(np.int32)
    ids = np.arange(nq, dtype=np.int64)[::-1].copy()
    s = SageScheduler(w, RoundConfig(k=32, theta=0.8, min_matches=20, max_len=2048, nbins=64))

    def pinned(a, off=0):
        # a pinned copy of a starting `off` bytes into a pinned block
        b = torch.empty(a.nbytes + 64, dtype=torch.uint8).pin_memory().numpy()
        v = b[off:off + a.nbytes].view(a.dtype).reshape(a.shape)
        v[:] = a
        return v

    ref_p, ref_G = s.schedule_round_host(q, qi, I, ids)  # pageable: copy-engine path
    ref_G, ref_p = ref_G.copy(), ref_p.copy()
    for off in (0, 4):
        for with_ids in (True, False):
            args = [pinned(q, off), pinned(qi, off), pinned(I, off), pinned(ids, 8 if off else 0)]
            if not with_ids:
                args[3] = None
            G = pinned(np.zeros(nq)); perm = pinned(np.zeros(nq, dtype=np.int64))
            for _ in range(3):  # eager, eager, captured replay
                G[:] = 0
                s.schedule_round_host(*args, G, perm)
                assert np.array_equal(G, ref_G), (off, with_ids)
                if with_ids:
                    assert np.array_equal(perm, ref_p), (off, with_ids)
                else:
                    assert np.array_equal(np.sort(perm), np.arange(nq))


def test_round_fallback_and_cold_start(cuda):
    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    w = HistoryWindow(64, 128)
    s = SageScheduler(w, RoundConfig(k=8, theta=0.99, nbins=64))
    q = np.ones((2, 128), np.int8)
    with pytest.raises(_lib.ColdStartError):
        s.predict(q, O.inv_norm(q), np.array([5, 6]))
    rng = np.random.default_rng(1)
    e = rng.integers(-5, 6, (40, 128)).astype(np.int8)
    L = rng.integers(1, 2049, 40).astype(np.int32)
    w.push(e, L)
    st = s.predict(q, O.inv_norm(q), np.array([5, 6]))
    assert st.used_fb.cpu().tolist() == [1, 1]  # nothing is >= 0.99 similar
    bins, c, D = O.hist_to_points(*O.bin_hist(L, 2048, 64), 5)
    assert np.array_equal(st.pcnt[0, :c.size].cpu().numpy(), c)
    assert st.G[0].item() == O.gittins_points(c, D)


def test_predict_dropin_limit_equals_reference_match(cuda):
    """predict() with k >= #matches and width-1 bins returns exactly the
    reference's threshold-match pmf (match_pmfs)."""
    from paper_2603_07917_b200.predictor import Request, SemanticHistory, predict
    w, be, bl, q, qi = _bank(2000, 128, 10, 3, 4)
    keys = O.scores(q, qi, be, O.inv_norm(be))
    for i in range(4):
        hits = np.flatnonzero(keys[i] >= np.float32(0.8))
        if hits.size > 256 or hits.size < 1:
            continue
        req = Request(id=i, prompt_tokens=np.arange(3), input_len=10)
        req.embedding, req.inv_norm = _t(q[i]), _t(qi[i:i + 1])[0]
        d = predict(SemanticHistory(theta=0.8, min_matches=1, k=256), req, w)
        sup = np.zeros((1, 2049))
        mas = np.zeros((1, 2049))
        sz = np.zeros(1, np.int64)
        O.match_pmfs(keys[i:i + 1], bl.astype(np.int64), np.float32(0.8), 2048, sup, mas, sz)
        assert np.array_equal(d.support, sup[0, :sz[0]])
        np.testing.assert_allclose(d.masses, mas[0, :sz[0]], rtol=1e-15, atol=0)


# ------------------------------------------------- refresh + rank (c3) -----
def _c3_laws(n, nbins, seed, P=None):
    rng = np.random.default_rng(seed)
    P = P or nbins
    I = rng.integers(1, 4097, n).astype(np.int32)
    npts = np.zeros(n, np.int32)
    pc = np.zeros((n, P), np.int32)
    pD = np.zeros((n, P), np.int64)
    for i in range(n):
        lens = rng.integers(1, 2049, 64) if i % 3 else np.clip(
            np.rint(np.exp(rng.normal(5, 0.7, 64))), 1, 2048).astype(np.int64)
        _, c, D = O.hist_to_points(*O.bin_hist(lens, 2048, nbins), I[i])
        npts[i] = c.size
        pc[i, :c.size] = c
        pD[i, :c.size] = D
    g = np.where(rng.random(n) < 0.4, rng.integers(0, 2049, n), 0).astype(np.int32)
    return I, npts, pc, pD, g


def test_refresh_bit_exact(cuda):
    from paper_2603_07917_b200 import _lib
    n, nbins = 3000, 512
    I, npts, pc, pD, g = _c3_laws(n, nbins, 4)
    bucket = np.zeros(n, np.int32)
    G = np.full(n, -1.0)
    dI, dg, db, dn, dpc, dpD, dG = map(_t, (I, g, bucket, npts, pc, pD, G))
    ref_flag = torch.zeros(n, dtype=torch.uint8, device="cuda")
    _lib.call("ss_refresh", n, dI.data_ptr(), dg.data_ptr(), db.data_ptr(), 200, dn.data_ptr(),
              dpc.data_ptr(), dpD.data_ptr(), nbins, dG.data_ptr(), ref_flag.data_ptr(), 1,
              _lib.stream_ptr())
    got = dG.cpu().numpy()
    for i in range(n):
        k = npts[i]
        ref = O.gittins_points(pc[i, :k], pD[i, :k], int(I[i]), int(g[i]))
        assert got[i] == ref, (i, got[i], ref)
    assert np.array_equal(db.cpu().numpy(), g // 200)
    # not due -> untouched
    dG.fill_(-1.0)
    _lib.call("ss_refresh", n, dI.data_ptr(), dg.data_ptr(), db.data_ptr(), 200, dn.data_ptr(),
              dpc.data_ptr(), dpD.data_ptr(), nbins, dG.data_ptr(), ref_flag.data_ptr(), 0,
              _lib.stream_ptr())
    assert (dG == -1.0).all() and int(ref_flag.sum()) == 0


@pytest.mark.parametrize("kv,mode", [(None, "cut"), (12_000, "cut"), (12_000, "skip")])
def test_c5_replay_rolling_inserts_bit_exact(cuda, kv, mode):
    """BASELINE configs[4] at test scale: trace replay with rolling bank inserts
    (completions evict the oldest records), admission predict, bucket
    refreshes and a full re-rank every round -- G and the order bit-exact vs an
    independent numpy replica of the same loop over the oracle."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.replay import Trace, replay
    from paper_2603_07917_b200.scheduler import RoundConfig
    cap, dim, ntr = 3000, 128, 1500
    emb, lens, _, _ = O.make_bank(cap + ntr, dim, 40, 77)
    rng = np.random.default_rng(78)
    tr = Trace(emb=emb[cap:], inv=O.inv_norm(emb[cap:]),
               input_len=rng.integers(1, 4097, ntr).astype(np.int32),
               true_len=np.clip(lens[cap:], 1, 600).astype(np.int32))
    cfg = RoundConfig(k=16, theta=0.8, min_matches=5, max_len=2048, nbins=64)
    A, TOK, B, R = 64, 40, 48, 30
    w = HistoryWindow(cap, dim)
    w.push(emb[:cap], lens[:cap])

    # ---- numpy replica ----
    bank_e = list(emb[:cap])
    bank_l = list(lens[:cap])
    st = {}  # rid -> dict(c, D, I, g, bucket, G)
    running = []
    nxt = 0
    expected = []
    for r in range(R):
        done = []
        for rid in running:
            st[rid]["g"] += TOK
            if st[rid]["g"] >= tr.true_len[rid]:
                done.append(rid)
        for rid in done:
            bank_e.append(tr.emb[rid])
            bank_l.append(tr.true_len[rid])
            del st[rid]
        bank_e, bank_l = bank_e[-cap:], bank_l[-cap:]
        head = cap + sum(1 for _ in ())  # seq only matters relatively
        n_new = min(A, ntr - nxt, 10_000)
        be = np.array(bank_e)
        bl = np.array(bank_l)
        seq = np.arange(len(bank_e))
        if n_new:
            ids = np.arange(nxt, nxt + n_new)
            keys = O.scores(tr.emb[ids], tr.inv[ids], be, O.inv_norm(be))
            res = O.predict_round(keys, seq, bl, tr.input_len[ids], cfg.k, cfg.theta,
                                  cfg.min_matches, cfg.max_len, cfg.nbins, window_lens=bl)
            for rid, x in zip(ids, res):
                st[int(rid)] = dict(c=x["c"], D=x["D"], I=int(tr.input_len[rid]), g=0, bucket=0,
                                    G=x["G"])
            nxt += n_new
        act = np.array(sorted(st), dtype=np.int64)
        for rid in act:
            s = st[int(rid)]
            if s["g"] // 200 > s["bucket"]:
                s["G"] = O.gittins_points(s["c"], s["D"], s["I"], s["g"])
                s["bucket"] = s["g"] // 200
        G = np.array([st[int(i)]["G"] for i in act])
        perm = O.rank(G, act)
        if kv is None:
            running = [int(act[p]) for p in perm[:B]]
        else:
            b, _ = O.pack_batch(perm, [st[int(i)]["I"] for i in act],
                                [st[int(i)]["g"] for i in act], kv, B, mode)
            running = [int(act[i]) for i in b]
        expected.append((act, G, perm, running))
        del head

    got = []
    stats = replay(w, tr, cfg, A, TOK, B, max_active=2048, rounds=R,
                   on_round=lambda r, info: got.append(info), kv_capacity=kv, pack_mode=mode)
    assert stats.completed > (50 if kv is None else 0) and stats.refreshed > (20 if kv is None else 0)
    assert len(got) == len(expected)
    for (act, G, perm, running), info in zip(expected, got):
        assert np.array_equal(info["active_ids"], act)
        assert np.array_equal(info["G"], G)
        assert np.array_equal(info["perm"], perm)
        assert info["running"] == running


def test_c3_refresh_storm_full_size(cuda):
    """BASELINE configs[2]: 200k running+pending requests, 512-bin cost laws
    (from 64 length draws each), index recompute + full re-rank.  Laws and G
    bit-exact on a 20k-request sample vs the oracle; the full ranking is
    exactly the (G, id) order of the 200k indices."""
    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.scheduler import rank
    n, nbins, k = 200_000, 512, 64
    rng = np.random.default_rng(31)
    lens = np.clip(np.rint(np.exp(rng.normal(5.5, 0.8, (n, k)))), 1, 2048).astype(np.int32)
    I = rng.integers(1, 4097, n).astype(np.int32)
    g = np.where(rng.random(n) < 0.4, rng.integers(0, 2049, n), 0).astype(np.int32)
    d = "cuda"
    comp = torch.ones((n, k), dtype=torch.int64, device=d)  # every draw is a "neighbour"
    fb = torch.zeros((3, nbins), dtype=torch.int64, device=d)
    npts = torch.zeros(n, dtype=torch.int32, device=d)
    pbin = torch.zeros((n, nbins), dtype=torch.int32, device=d)
    pcnt = torch.zeros((n, nbins), dtype=torch.int32, device=d)
    pD = torch.zeros((n, nbins), dtype=torch.int64, device=d)
    G = torch.zeros(n, dtype=torch.float64, device=d)
    dl, dI, dg = _t(lens), _t(I), _t(g)
    P = lambda t: t.data_ptr()  # noqa: E731
    _lib.call("ss_finish", P(comp), P(dl), n, k, 1, 2048, nbins, P(dI), P(fb[0]), P(fb[1]),
              P(fb[2]), nbins, P(npts), P(pbin), P(pcnt), P(pD), None, None, P(G),
              _lib.stream_ptr())
    bucket = torch.zeros(n, dtype=torch.int32, device=d)
    _lib.call("ss_refresh", n, P(dI), P(dg), P(bucket), 200, P(npts), P(pcnt), P(pD), nbins,
              P(G), None, 1, _lib.stream_ptr())
    ids = _t(np.arange(n, dtype=np.int64))
    perm = rank(G, ids).cpu().numpy()
    Gh = G.cpu().numpy()
    assert np.array_equal(perm, O.rank(Gh, np.arange(n)))
    sample = rng.choice(n, 20_000, replace=False)
    np_, pc, pd_ = npts.cpu().numpy(), pcnt.cpu().numpy(), pD.cpu().numpy()
    for i in sample:
        bins, c, D = O.hist_to_points(*O.bin_hist(lens[i], 2048, nbins), I[i])
        assert np_[i] == c.size
        assert np.array_equal(pc[i, :c.size], c) and np.array_equal(pd_[i, :c.size], D)
        assert Gh[i] == O.gittins_points(c, D, int(I[i]), int(g[i])), i


@pytest.mark.parametrize("n", [1, 7, 1024, 4096, 4097, 5120, 5121, 6000, 8192, 8193, 20_000, 200_000, 1_000_003])
def test_rank_bit_exact(cuda, n):
    from paper_2603_07917_b200.scheduler import rank
    rng = np.random.default_rng(n)
    G = rng.choice(rng.uniform(1, 1e7, max(2, n // 3)), n)  # many exact ties
    ids = rng.permutation(n).astype(np.int64)
    perm = rank(_t(G), _t(ids)).cpu().numpy()
    assert np.array_equal(perm, O.rank(G, ids))
    perm = rank(_t(G)).cpu().numpy()
    assert np.array_equal(perm, O.rank(G, np.arange(n)))
    # ascending ids (the onesweep skips its id passes) with gaps
    sids = np.cumsum(rng.integers(1, 5, n)).astype(np.int64)
    perm = rank(_t(G), _t(sids)).cpu().numpy()
    assert np.array_equal(perm, O.rank(G, sids))


@pytest.mark.parametrize("n", [3001, 7001, 50_000])
def test_rank_special_values(cuda, n):
    """inf (no law yet), zero, wide exponent range, negative and > 2^32 ids
    (counting rank and onesweep)."""
    from paper_2603_07917_b200.scheduler import rank
    rng = np.random.default_rng(9)
    G = rng.choice(np.array([np.inf, 0.0, 1e-300, 1e300, 2.0, 2.0, 5e3, 7.25]), n)
    ids = rng.integers(-(1 << 40), 1 << 40, n).astype(np.int64)
    ids[:10] = ids[10]  # duplicate ids: index order breaks the tie (stable)
    perm = rank(_t(G), _t(ids)).cpu().numpy()
    assert np.array_equal(perm, np.lexsort((np.arange(n), ids, G)))


# ---------------------------------------------------- sharded round (N=1) ---
@pytest.mark.parametrize("owner", [0, None])
@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
def test_sharded_round_world1_equals_single_gpu(cuda, exchange, owner):
    """The multi-GPU round run as a 1-rank NCCL group equals the fused
    single-GPU round bit for bit: single owner (query broadcast, local top-k,
    candidate all-gather or the fused P2P gather, merge, histogram
    all-reduce) and per-rank queues (query all-gather, all-to-all or P2P
    scatter).  The host-buffer call is replayed from its captured graph, and
    a push between two host calls (the ring head moves) is honoured."""
    import socket

    import torch.distributed as dist

    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.sharded import ShardedHistory, ShardedScheduler
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda:0"))
    try:
        n, dim, nq, extra = 20_000, 384, 200, 300
        emb, lens, _, _ = O.make_bank(n + nq + extra, dim, 50, 9)
        cfg = RoundConfig(k=32, theta=0.8, nbins=64)
        sh = ShardedHistory(n, dim)
        sh.push(torch.as_tensor(emb[:n], device="cuda"), torch.as_tensor(lens[:n], device="cuda"))
        q, qi = emb[n:n + nq], O.inv_norm(emb[n:n + nq])
        I = np.random.default_rng(0).integers(1, 4097, nq).astype(np.int32)
        ids = np.arange(nq)
        ss = ShardedScheduler(sh, cfg, exchange=exchange, owner=owner)
        p1, G1, _ = ss.schedule_round(_t(q), _t(qi), _t(I), _t(ids))
        p1, G1 = p1.clone(), G1.clone()
        # the host-buffer call (captured round + copies), twice: same answer
        hG = torch.empty(nq, dtype=torch.float64).pin_memory()
        hp = torch.empty(nq, dtype=torch.int64).pin_memory()
        for _ in range(2):
            hG.zero_()
            hp.zero_()
            ss.schedule_round_host(q, qi, I, ids.astype(np.int64), hG, hp)
            assert torch.equal(hG, G1.cpu()) and torch.equal(hp, p1.cpu())
        if ss.peer is not None:
            p1b, G1b, _ = ss.schedule_round(_t(q), _t(qi), _t(I), _t(ids))  # buffers reused
            assert torch.equal(G1b, G1) and torch.equal(p1b, p1)
        w = HistoryWindow(n, dim)
        w.push(emb[:n], lens[:n])
        p0, G0, _ = SageScheduler(w, cfg).schedule_round(_t(q), _t(qi), _t(I), _t(ids))
        assert torch.equal(G1, G0) and torch.equal(p1, p0)
        # rolling inserts (wrap the ring by `extra` rows, identical prompts
        # among them so the insertion_seq tie rule matters): the host call
        # re-captures for the new head and still equals the single-GPU round
        new_e = emb[n + nq:n + nq + extra].copy()
        new_e[: nq // 2] = q[: nq // 2]  # exact duplicates of queries -> ties on cos 1.0
        new_l = lens[n + nq:n + nq + extra]
        sh.push(torch.as_tensor(new_e, device="cuda"), torch.as_tensor(new_l, device="cuda"))
        w.push(new_e, new_l)
        hG.zero_()
        ss.schedule_round_host(q, qi, I, ids.astype(np.int64), hG, hp)
        p2, G2, _ = SageScheduler(w, cfg).schedule_round(_t(q), _t(qi), _t(I), _t(ids))
        assert torch.equal(hG, G2.cpu()) and torch.equal(hp, p2.cpu())
        if ss.peer is not None:
            ss.peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_topk_gather_shards_equal_single_bank(cuda, world):
    """ss_topk_gather addressing (single-owner exchange), all ranks simulated
    in one process: every shard stores its merged rows for the owner's whole
    queue at [r][q] of the owner's buffer; merging that buffer gives the
    single-bank top-k, lengths included, bit for bit."""
    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.sharded import ShardPlan
    n, dim, nq, k = 9_000, 384, 150, 32
    emb, lens, _, _ = O.make_bank(n + nq, dim, 40, 6)
    q = _t(emb[n:])
    qi = _t(O.inv_norm(emb[n:]))
    recv_c = torch.full((world, nq, k), -7, dtype=torch.int64, device="cuda")
    recv_l = torch.full((world, nq, k), -7, dtype=torch.int32, device="cuda")
    for r in range(world):
        plan = ShardPlan(n, world, r)
        w = HistoryWindow(plan.local_capacity, dim, global_capacity=n, slot_offset=plan.slot_offset)
        idx, seq, slot = plan.route(0, n)
        w.write(_t(emb[idx]), _t(lens[idx]), _t(seq), _t(slot))
        w.set_head(n)
        _lib.call("ss_topk_gather", w.handle, _lib.ptr(q), _lib.ptr(qi), nq, k, 0.6, 0, world, r,
                  _lib.ptr(recv_c), _lib.ptr(recv_l), _lib.stream_ptr())
    out_c = torch.empty((nq, k), dtype=torch.int64, device="cuda")
    out_l = torch.empty((nq, k), dtype=torch.int32, device="cuda")
    _lib.call("ss_merge_topk", _lib.ptr(recv_c), _lib.ptr(recv_l), world, nq, k,
              _lib.ptr(out_c), _lib.ptr(out_l), _lib.stream_ptr())
    full, *_ = _bank(n, dim, 40, 6, nq)
    c0, l0 = full.topk(q, qi, k, 0.6)
    assert torch.equal(out_c, c0) and torch.equal(out_l, l0)


@pytest.mark.parametrize("nlists,k,fill", [(8, 64, "full"), (8, 64, "ragged"), (3, 20, "ragged"),
                                            (18, 64, "ragged"), (8, 256, "full"), (1, 64, "ragged"),
                                            (40, 64, "full"), (5, 7, "empty")])
def test_merge_topk_vs_sorted_union(cuda, nlists, k, fill):
    """ss_merge_topk (the owner's merge of the shards' lists; the warp-per-query
    kernel up to nlists * k = 2048 candidates, the block kernel above) against
    the sorted union of the lists: top-k composites descending, 0-padded, each
    with its carried length.  Keys tie across lists (same high word, different
    insertion rank) so the low-word resolution is exercised; lists are in
    arbitrary order and partly empty."""
    from paper_2603_07917_b200 import _lib
    rng = np.random.default_rng(nlists * 1000 + k)
    nq = 300
    pool = nlists * k
    comp = np.zeros((nlists, nq, k), np.uint64)
    ln = np.zeros((nlists, nq, k), np.int32)
    for q in range(nq):
        keys = rng.integers(0x3F000000, 0x3F000000 + max(4, pool // 3), pool).astype(np.uint64)
        rel = rng.permutation(1 << 20)[:pool].astype(np.uint64)  # unique insertion ranks
        c = (keys << np.uint64(32)) | rel
        for l in range(nlists):
            n = {"full": k, "ragged": int(rng.integers(0, k + 1)), "empty": 0}[fill]
            part = c[l * k:l * k + n]
            comp[l, q, :n] = rng.permutation(part)
            ln[l, q, :n] = (part % np.uint64(2047)).astype(np.int32) + 1
    out_c = torch.full((nq, k), -5, dtype=torch.int64, device="cuda")
    out_l = torch.full((nq, k), -5, dtype=torch.int32, device="cuda")
    dc, dl = _t(comp.view(np.int64)), _t(ln)
    _lib.call("ss_merge_topk", _lib.ptr(dc), _lib.ptr(dl), nlists, nq, k, _lib.ptr(out_c),
              _lib.ptr(out_l), _lib.stream_ptr())
    got_c = out_c.cpu().numpy().view(np.uint64)
    got_l = out_l.cpu().numpy()
    for q in range(nq):
        allc = comp[:, q, :].ravel()
        alll = ln[:, q, :].ravel()
        nz = allc != 0
        order = np.argsort(allc[nz])[::-1][:k]
        want_c = np.zeros(k, np.uint64)
        want_l = np.zeros(k, np.int32)
        want_c[:order.size] = allc[nz][order]
        want_l[:order.size] = alll[nz][order]
        assert np.array_equal(got_c[q], want_c), q
        assert np.array_equal(got_l[q], want_l), q


@pytest.mark.parametrize("world,algo", [(2, "auto"), (3, "auto"), (2, "scan")])
def test_topk_scatter_shards_equal_single_bank(cuda, world, algo):
    """ss_topk_scatter addressing, all ranks simulated in one process: shard r
    stores the merged rows of every rank's queries into that rank's receive
    buffer at [r][q]; merging a receive buffer gives the single-bank top-k of
    the owner's queries (lengths included), bit for bit."""
    import ctypes as C

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.sharded import ShardPlan
    n, dim, nq, k = 6_000, 384, 70, 16
    emb, lens, _, _ = O.make_bank(n + world * nq, dim, 40, 5)
    q = _t(emb[n:])
    qi = _t(O.inv_norm(emb[n:]))
    wins = []
    for r in range(world):
        plan = ShardPlan(n, world, r)
        w = HistoryWindow(plan.local_capacity, dim, global_capacity=n, slot_offset=plan.slot_offset)
        idx, seq, slot = plan.route(0, n)
        w.write(_t(emb[idx]), _t(lens[idx]), _t(seq), _t(slot))
        w.set_head(n)
        wins.append(w)
    recv_c = [torch.full((world, nq, k), -7, dtype=torch.int64, device="cuda") for _ in range(world)]
    recv_l = [torch.full((world, nq, k), -7, dtype=torch.int32, device="cuda") for _ in range(world)]
    tc = (C.c_void_p * world)(*[t.data_ptr() for t in recv_c])
    tl = (C.c_void_p * world)(*[t.data_ptr() for t in recv_l])
    for r, w in enumerate(wins):
        _lib.call("ss_topk_scatter", w.handle, _lib.ptr(q), _lib.ptr(qi), world * nq, k, 0.5,
                  _lib.ALGO[algo], world, r, tc, tl, _lib.stream_ptr())
    full, *_ = _bank(n, dim, 40, 5, world * nq)
    c0, l0 = full.topk(q, qi, k, 0.5)
    for r in range(world):
        out_c = torch.empty((nq, k), dtype=torch.int64, device="cuda")
        out_l = torch.empty((nq, k), dtype=torch.int32, device="cuda")
        _lib.call("ss_merge_topk", _lib.ptr(recv_c[r]), _lib.ptr(recv_l[r]), world, nq, k,
                  _lib.ptr(out_c), _lib.ptr(out_l), _lib.stream_ptr())
        assert torch.equal(out_c, c0[r * nq:(r + 1) * nq])
        assert torch.equal(out_l, l0[r * nq:(r + 1) * nq])
    with pytest.raises(ValueError):
        _lib.call("ss_topk_scatter", wins[0].handle, _lib.ptr(q), _lib.ptr(qi), world * nq - 1, k,
                  0.5, 0, world, 0, tc, tl, _lib.stream_ptr())


@pytest.mark.parametrize("mode", ["owner", "per-rank", "owner-coll"])
def test_sharded_p2p_two_ranks_one_gpu(cuda, mode):
    """World-2 round, two processes on cuda:0 (tests/_p2p_worker.py), with the
    fused P2P merge + exchange or (owner-coll) the collective exchange: the
    queue owner's result equals the single-GPU round (single owner: rank 1
    holds the whole queue)."""
    import pathlib
    import socket
    import subprocess
    import sys
    root = pathlib.Path(__file__).resolve().parents[1]
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node=2", "--master-addr=127.0.0.1", f"--master-port={port}",
                        str(root / "tests" / "_p2p_worker.py"), mode], cwd=str(root),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])


def test_ipc_buffer_cross_process(cuda, tmp_path):
    """ss_ipc_malloc/handle in this process, ss_ipc_open + stores in another
    (the mapping the P2P exchange uses between ranks of a node)."""
    import ctypes as C
    import subprocess
    import sys

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import _cuda_view
    p = C.c_void_p()
    _lib.call("ss_ipc_malloc", 0, 4096 * 8, C.byref(p))
    try:
        h = (C.c_uint8 * 64)()
        _lib.call("ss_ipc_handle", p, h)
        child = (
            "import ctypes as C, torch\n"
            "from paper_2603_07917_b200 import _lib\n"
            "from paper_2603_07917_b200.history import _cuda_view\n"
            "torch.cuda.init()\n"
            f"h = (C.c_uint8 * 64).from_buffer_copy(bytes.fromhex('{bytes(h).hex()}'))\n"
            "p = C.c_void_p()\n"
            "_lib.call('ss_ipc_open', h, C.byref(p))\n"
            "t = _cuda_view(p.value, torch.int64, (4096,), 0)\n"
            "t.copy_(torch.arange(4096, device='cuda') * 3 + 1)\n"
            "torch.cuda.synchronize()\n"
            "_lib.call('ss_ipc_close', p)\n")
        r = subprocess.run([sys.executable, "-c", child], cwd=str(__import__("pathlib").Path(__file__).resolve().parents[1]), capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        got = _cuda_view(p.value, torch.int64, (4096,), 0).cpu()
        assert torch.equal(got, torch.arange(4096) * 3 + 1)
    finally:
        _lib.call("ss_ipc_free", p)


# ------------------------------------------- batch formation --
@pytest.mark.parametrize("mode", ["cut", "skip"])
@pytest.mark.parametrize("n,K,B", [(0, 8192, 64), (1, 8192, 64), (7, 20, 3), (1024, 8192, 64),
                                   (3000, 60_000, 2000), (5000, 8192, 4096),
                                   (200_000, 8192, 64), (200_000, 1 << 40, 5000),
                                   (20_000, 1 << 40, 20_000), (9000, 5_000_000, 9000)])
def test_pack_batch_bit_exact(cuda, mode, n, K, B):
    from paper_2603_07917_b200.scheduler import pack_batch
    rng = np.random.default_rng(n + B)
    Imax = min(4096, K - 1)
    I = rng.integers(1, Imax + 1, n).astype(np.int32)
    running = rng.random(n) < 0.4
    g = np.where(running, rng.integers(0, 2049, n), 0).astype(np.int32)
    perm = rng.permutation(n).astype(np.int64)
    plan = pack_batch(_t(perm), _t(I), _t(g), K, B, mode)
    batch, tokens = plan.host()
    ref, ref_tokens = O.pack_batch(perm, I, g, K, B, mode)
    assert batch.tolist() == ref and tokens == ref_tokens


def test_pack_batch_cannot_fit(cuda):
    from paper_2603_07917_b200.scheduler import pack_batch
    I = np.array([5, 9000, 7, 9001], np.int32)
    plan = pack_batch(_t(np.arange(4)), _t(I), _t(np.zeros(4, np.int32)), 8192, 64)
    with pytest.raises(ValueError, match="request 1 cannot fit"):
        plan.host()


def test_trace_to_replay(cuda, tmp_path):
    """Generated JSONL trace -> GPU feature-hash embedding (bit-exact vs the
    reference hash) -> replay with KV-packed batches."""
    from paper_2603_07917_b200.history import DEFAULT_SALT, HistoryWindow
    from paper_2603_07917_b200.replay import replay
    from paper_2603_07917_b200.scheduler import RoundConfig
    from paper_2603_07917_b200.trace import (ClusterSpec, LengthLaw, WorkloadConfig,
                                             generate_trace, load_trace, save_trace,
                                             to_replay_trace)
    rng = np.random.default_rng(5)
    cl = tuple(ClusterSpec(tuple(int(x) for x in rng.integers(0, 50_000, 40)), 6,
                           LengthLaw("lognormal", (float(rng.uniform(3, 6)), 0.5)))
               for _ in range(12))
    reqs = generate_trace(WorkloadConfig(lam=10.0, n_requests=1200, clusters=cl, seed=2))
    f = tmp_path / "t.jsonl"
    save_trace(reqs, str(f))
    tr = to_replay_trace(load_trace(str(f)), dim=384)
    ref = np.stack([O.embed_accumulate(r.prompt_tokens, DEFAULT_SALT, 384) for r in reqs[:50]])
    assert np.array_equal(tr.emb[:50], ref.astype(np.int8))
    w = HistoryWindow(400, 384)
    w.push(tr.emb[:400], tr.true_len[:400], tr.inv[:400])
    cfg = RoundConfig(k=16, theta=0.8, min_matches=5, max_len=2048, nbins=64)
    batches = []
    st = replay(w, tr, cfg, 50, 32, 64, max_active=1024, rounds=20,
                on_round=lambda r, info: batches.append(info["running"]), kv_capacity=8192,
                pack_mode="skip")
    assert st.rounds == 20 and st.admitted == 1000
    assert all(sum(tr.input_len[i] for i in b) <= 8192 for b in batches)


@pytest.mark.parametrize("kv,mode", [(None, "cut"), (12_000, "skip")])
def test_c5_device_replay_equals_host_replay(cuda, kv, mode):
    """The device-resident replay (bench --config c5) reproduces the host
    driver (checked above against the numpy replica) round by round."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.replay import Trace, replay
    from paper_2603_07917_b200.replay_device import DeviceReplay, DeviceTrace
    from paper_2603_07917_b200.scheduler import RoundConfig
    cap, dim, ntr = 3000, 128, 2500
    emb, lens, _, _ = O.make_bank(cap + ntr, dim, 40, 91)
    rng = np.random.default_rng(92)
    tr = Trace(emb=emb[cap:], inv=O.inv_norm(emb[cap:]),
               input_len=rng.integers(1, 4097, ntr).astype(np.int32),
               true_len=np.clip(lens[cap:], 1, 500).astype(np.int32))
    cfg = RoundConfig(k=16, theta=0.8, min_matches=5, max_len=2048, nbins=64)
    A, TOK, B, R, MAXA = 80, 48, 64, 40, 700
    w1 = HistoryWindow(cap, dim)
    w1.push(emb[:cap], lens[:cap])
    host = []
    replay(w1, tr, cfg, A, TOK, B, max_active=MAXA, rounds=R,
           on_round=lambda r, info: host.append(info), kv_capacity=kv, pack_mode=mode)
    w2 = HistoryWindow(cap, dim)
    w2.push(emb[:cap], lens[:cap])
    dr = DeviceReplay(w2, DeviceTrace.from_host(tr), cfg, A, TOK, B, MAXA, kv, mode)
    dev = []
    for _ in range(R):
        out = dr.round()
        if dr.n_act:
            dev.append(dr.info(out["perm"]))
    assert len(dev) == len(host) and dr.stats.completed > 50
    assert dr.stats.refreshed > (20 if kv is None else 0)
    for a, b in zip(host, dev):
        assert np.array_equal(a["active_ids"], b["active_ids"])
        assert np.array_equal(a["G"][:a["active_ids"].size], b["G"])
        assert np.array_equal(a["perm"], b["perm"])
        assert a["running"] == b["running"]
    # the rings saw the same pushes in the same order
    e1, i1, l1, s1 = w1.tensors()
    e2, i2, l2, s2 = w2.tensors()
    assert w1.head == w2.head and torch.equal(s1, s2) and torch.equal(l1, l2) and torch.equal(e1, e2)


@pytest.mark.parametrize("dim", [128, 256, 512])
@pytest.mark.parametrize("nq", [64, 300])
def test_topk_dims_bit_exact(cuda, dim, nq):
    """Other embedding widths through the tcgen05 kernels (dim 512 leaves
    room for only the N=192 double buffer beside A in TMEM)."""
    w, be, bl, q, qi = _bank(12_000, dim, 60, 17, nq)
    for theta, k in ((0.8, 64), (-1.0, 32)):
        keys, seq, ref = _oracle_topk(w, be, q, qi, k, theta)
        comp, ln = w.topk(q, qi, k, theta, "tcgen05")
        _check_topk(w, comp, keys, seq, ref, k)


@pytest.mark.parametrize("kv,mode", [(None, "cut"), (12_000, "skip")])
def test_c5_native_engine_equals_device_replay(cuda, kv, mode):
    """ss_engine_round (one native call per round) reproduces the torch-driven
    device replay round by round, including the ring it leaves behind."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.replay import Trace
    from paper_2603_07917_b200.replay_device import DeviceReplay, DeviceTrace, NativeReplay
    from paper_2603_07917_b200.scheduler import RoundConfig
    cap, dim, ntr = 3000, 128, 2500
    emb, lens, _, _ = O.make_bank(cap + ntr, dim, 40, 93)
    rng = np.random.default_rng(94)
    tr = Trace(emb=emb[cap:], inv=O.inv_norm(emb[cap:]),
               input_len=rng.integers(1, 4097, ntr).astype(np.int32),
               true_len=np.clip(lens[cap:], 1, 500).astype(np.int32))
    dtr = DeviceTrace.from_host(tr)
    cfg = RoundConfig(k=16, theta=0.8, min_matches=5, max_len=2048, nbins=64)
    A, TOK, B, R, MAXA = 80, 48, 64, 40, 700
    w1 = HistoryWindow(cap, dim)
    w1.push(emb[:cap], lens[:cap])
    w2 = HistoryWindow(cap, dim)
    w2.push(emb[:cap], lens[:cap])
    ref = DeviceReplay(w1, dtr, cfg, A, TOK, B, MAXA, kv, mode)
    nat = NativeReplay(w2, dtr, cfg, A, TOK, B, MAXA, kv, mode)
    for r in range(R):
        out = ref.round()
        nat.round()
        assert nat.n_act == ref.n_act, r
        if ref.n_act:
            a, b = ref.info(out["perm"]), nat.info()
            assert np.array_equal(a["active_ids"], b["active_ids"]), r
            assert np.array_equal(a["G"], b["G"]), r
            assert np.array_equal(a["perm"], b["perm"]), r
            assert a["running"] == b["running"], r
    assert nat.stats.completed == ref.stats.completed > 50
    e1, i1, l1, s1 = w1.tensors()
    e2, i2, l2, s2 = w2.tensors()
    assert w1.head == w2.head and torch.equal(s1, s2) and torch.equal(l1, l2) and torch.equal(e1, e2)
    assert torch.equal(i1.view(torch.int32), i2.view(torch.int32))


def test_overhead_budget_spec(cuda):
    """SPEC.md:597 overhead budget: a full predict+priority pass over a queue
    of 1,000 requests (10,000-record window) completes in < 50 ms mean, and
    1,000 -> 2,000 queue entries grows the latency by less than 2.5x.  Timed
    through the host-buffer plugin call (copies and sync included)."""
    import time
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    emb, lens, _, _ = O.make_bank(10_000 + 2000, 384, 100, 31)
    w = HistoryWindow(10_000, 384)
    w.push(emb[:10_000], lens[:10_000])
    s = SageScheduler(w, RoundConfig(k=64, theta=0.8, min_matches=20, max_len=2048, nbins=128))
    rng = np.random.default_rng(5)

    def mean_ms(nq, reps=20):
        q = emb[10_000:10_000 + nq]
        qi, I, ids = O.inv_norm(q), rng.integers(1, 4097, nq).astype(np.int32), np.arange(nq)
        s.schedule_round_host(q, qi, I, ids)  # warm-up (workspace growth)
        t0 = time.perf_counter()
        for _ in range(reps):
            s.schedule_round_host(q, qi, I, ids)
        return (time.perf_counter() - t0) / reps * 1e3

    t1, t2 = mean_ms(1000), mean_ms(2000)
    assert t1 < 50.0, t1
    assert t2 < 2.5 * t1 + 0.5, (t1, t2)  # +0.5 ms slack: both are sub-millisecond here


def test_c2_round_time_guard(cuda):
    """Performance guard on BASELINE configs[1] (1M-row bank, 1024 requests,
    theta 0.8): the graph-replayed round stays under 0.6 ms (measured
    0.39-0.41 ms across boxes; a regression such as the similarity kernel's
    chunk registers spilling to local memory shows up as ~0.6 ms)."""
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries
    emb, lens, _ = make_bank_device(1 << 20, 384, 4096, 0)
    w = HistoryWindow(1 << 20, 384)
    w.push(emb, lens)
    del emb, lens
    q, qi, I, ids = make_queries(1024, 384, 4096, 0, qseed=1000)
    s = SageScheduler(w, RoundConfig(k=64, theta=0.8, min_matches=20, max_len=2048, nbins=128))
    g, _ = s.capture_round(_t(q), _t(qi), _t(I), _t(ids))
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    assert ms < 0.6, ms


def test_sharded_owner_stages_bit_identical_small(cuda):
    """The measured-component projection of the single-owner round
    (bench.c4_projection) at a small shape: the bank cut by ShardPlan into 2
    and 4 shards, each shard's local top-k, the owner's ss_merge_topk +
    ss_finish + ss_rank -- lists, window histogram, G and order bit-identical
    to the one-window round."""
    import bench
    out = bench.c4_projection(rows=1 << 16, nq=512, worlds=(2, 4), reps=1)
    assert [p["n_gpus"] for p in out["points"]] == [2, 4]
    assert all(p["bit_identical_to_one_gpu_round"] for p in out["points"])

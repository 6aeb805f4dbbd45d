"""Pin the CPU oracle: against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py) and against the SPEC's own known
answers.  CPU only."""

import numpy as np
import pytest

from oracle import sagesched_oracle as O


def test_match_pmfs_matches_reference_numba(golden):
    g = golden
    nq = g["mp_sims"].shape[0]
    sup = np.zeros_like(g["mp_sup"])
    mas = np.zeros_like(g["mp_mas"])
    sizes = np.zeros(nq, np.int64)
    O.match_pmfs(g["mp_sims"], g["mp_lens"], g["mp_theta"], int(g["mp_max_len"]), sup, mas, sizes)
    assert np.array_equal(sizes, g["mp_sizes"])
    for q in range(nq):
        k = sizes[q]
        assert np.array_equal(sup[q, :k], g["mp_sup"][q, :k])
        assert np.array_equal(mas[q, :k], g["mp_mas"][q, :k])  # bit-exact masses
    assert sizes[3] == 0  # zero-match query


def test_gittins_min_matches_reference(golden):
    g = golden
    for i in range(g["gm_value"].size):
        k = int(g["gm_npts"][i])
        v = O.gittins_min(g["gm_support"][i, :k], g["gm_masses"][i, :k])
        assert v == g["gm_value"][i]


def test_embed_matches_reference(golden):
    g = golden
    offs = g["em_offsets"]
    for d in (384, 256, 17):
        for i in range(offs.size - 1):
            v = O.embed_accumulate(g["em_tokens"][offs[i]:offs[i + 1]], int(g["em_salt"]), d)
            assert np.array_equal(v, g[f"em_{d}"][i])


def test_cost_matches_reference(golden):
    g = golden
    assert np.array_equal(O.cost_rb(g["cost_I"], g["cost_O"]), g["cost_rb"])
    rem = O.cost_rb(g["cost_I"], g["cost_O"]) - O.cost_rb(g["cost_I"], g["cost_o"])
    assert np.array_equal(rem, g["cost_rem"])
    for i in range(g["cd_n"].size):
        k = int(g["cd_n"][i])
        out = O.cost_vector("resource-bound", g["cd_I"][i], g["cd_sup"][i, :k])
        assert np.array_equal(out, g["cd_out"][i, :k])


# ---------------------------------------------------------------- App. A ----
@pytest.mark.parametrize("c", [1.0, 5.0, 1000.0])
def test_gittins_point_mass(c):
    assert O.gittins_min([c], [1.0]) == c


def test_gittins_bimodal_exact():
    assert O.gittins_min([1.0, 9.0], [0.5, 0.5]) == 2.0


def test_gittins_leading_zero_mass_raises():
    with pytest.raises(ZeroDivisionError):
        O.gittins_min([1.0, 2.0], [0.0, 1.0])


def test_gittins_support_point_min_equals_dense_grid():
    # 1000 random 2-10 point laws, grid step 1e-3*range
    rng = np.random.default_rng(0)
    for _ in range(1000):
        k = int(rng.integers(2, 11))
        s = np.sort(rng.choice(np.arange(1, 1000), k, replace=False)).astype(float)
        m = rng.dirichlet(np.ones(k))
        g = O.gittins_min(s, m)
        grid = O.gittins_dense_grid(s, m)
        assert grid >= g * (1 - 1e-9)
        assert g <= np.dot(s, m) * (1 + 1e-12)  # G <= mean
        assert abs(O.gittins_min(3.5 * s, m) - 3.5 * g) <= 1e-9 * g  # scale


def test_conditioning_examples():
    s, m = O.condition_on_attained([1.0, 9.0], [0.5, 0.5], 1.0)
    assert np.array_equal(s, [8.0]) and np.array_equal(m, [1.0])
    assert O.gittins_min(s, m) == 8.0
    s, m = O.condition_on_attained([2.0, 4.0, 8.0], [0.25, 0.25, 0.5], 3.0)
    assert np.allclose(s, [1.0, 5.0]) and np.allclose(m, [1 / 3, 2 / 3])
    # cond(cond(d, a), b) == cond(d, a + b)
    s1, m1 = O.condition_on_attained(*O.condition_on_attained([2.0, 4.0, 8.0, 16.0],
                                                              [0.1, 0.2, 0.3, 0.4], 3.0), 2.0)
    s2, m2 = O.condition_on_attained([2.0, 4.0, 8.0, 16.0], [0.1, 0.2, 0.3, 0.4], 5.0)
    assert np.allclose(s1, s2, atol=1e-9) and np.allclose(m1, m2, atol=1e-9)


def test_refresh_examples():
    assert O.refresh_due(199, 200)
    assert not O.refresh_due(200, 399)
    assert O.refresh_due(150, 650)


def test_cost_examples():
    assert O.cost_rb(100, 200) == 40000
    assert O.cost_rb(100, 200) - O.cost_rb(100, 100) == 25000
    out = O.cost_vector("resource-bound", 100, [100.0, 300.0])
    assert np.array_equal(out, [15000.0, 75000.0])
    assert O.cost_rb(5000, 10) > O.cost_rb(10, 50)


def test_integer_gittins_equals_reference_form():
    """The exact integer-count form (used on GPU) equals gittins_min on the
    mass form to ~1 ulp, with and without conditioning."""
    rng = np.random.default_rng(5)
    for _ in range(300):
        lens = rng.integers(1, 2049, int(rng.integers(1, 65)))
        I = int(rng.integers(1, 4097))
        for nbins in (64, 128, 512, 2048):
            bins, c, D = O.hist_to_points(*O.bin_hist(lens, 2048, nbins), I)
            s = O.points_support(c, D)
            m = c / c.sum()
            ref = O.gittins_min(s, m)
            assert abs(O.gittins_points(c, D) - ref) <= 1e-12 * ref
            g = int(rng.integers(0, 2048))
            a = g * g / 2 + I * g
            cond = O.condition_on_attained(s, m, a)
            got = O.gittins_points(c, D, I, g)
            if cond is None:
                assert got == ((g + 200) ** 2 - g * g) / 2 + I * 200
            else:
                ref = O.gittins_min(*cond)
                assert abs(got - ref) <= 1e-9 * ref


def test_predictor_examples_and_limit_reduction(golden):
    # 100 identical records of length 50 -> {50: 1}
    bins, c, D = O.hist_to_points(*O.bin_hist(np.full(100, 50), 2048, 2048), 7)
    assert np.array_equal(bins + 1, [50]) and np.array_equal(c, [100])
    # {1, 9} x 5 -> {1: .5, 9: .5}
    bins, c, D = O.hist_to_points(*O.bin_hist([1] * 5 + [9] * 5, 2048, 2048), 7)
    assert np.array_equal(bins + 1, [1, 9]) and np.array_equal(c / c.sum(), [0.5, 0.5])
    # limit k >= #matches, bin width 1 -> exactly reference match_pmfs
    g = golden
    sims, lens, theta, ml = g["mp_sims"], g["mp_lens"].copy(), g["mp_theta"], int(g["mp_max_len"])
    keep = lens >= 1
    for q in range(sims.shape[0]):
        hit = np.flatnonzero((sims[q] >= theta) & keep)
        sel = O.select_topk(sims[q][keep], np.arange(keep.sum()), 10**9, theta)
        assert sel.size == hit.size
        if hit.size == 0:
            continue
        bins, c, _ = O.hist_to_points(*O.bin_hist(lens[hit], ml, ml), 1)
        ref_sup = np.zeros(ml + 1)
        ref_mas = np.zeros(ml + 1)
        sz = np.zeros(1, np.int64)
        O.match_pmfs(sims[q:q + 1][:, keep], lens[keep], theta, ml, ref_sup[None], ref_mas[None], sz)
        assert np.array_equal(bins + 1.0, ref_sup[:sz[0]])
        assert np.allclose(c / c.sum(), ref_mas[:sz[0]], rtol=0, atol=1e-15)


def test_select_tie_break_larger_seq():
    keys = np.array([0.9, 0.95, 0.9, 0.9], np.float32)
    seq = np.array([10, 11, 30, 20])
    assert list(O.select_topk(keys, seq, 3, 0.8)) == [1, 2, 3]


def test_rank_examples():
    # bimodal {1,9} (G=2) beats deterministic {5} (G=5)
    G = [O.gittins_min([5.0], [1.0]), O.gittins_min([1.0, 9.0], [0.5, 0.5])]
    assert list(O.rank(G, [0, 1])) == [1, 0]
    # ties -> id order
    assert list(O.rank([3.0, 3.0, 1.0], [7, 2, 9])) == [2, 1, 0]


# ------------------------------------------- batch formation --
def test_pack_batch_spec_examples():
    from oracle import sagesched_oracle as O
    # K = I1 + 1 exactly, two identical pending requests -> strictly serial
    # (SPEC engine example "capacity forces serialization")
    assert O.pack_batch([0, 1], [10, 10], [0, 0], 11, 64) == ([0], 11)
    # count limit B
    assert O.pack_batch(range(5), [1] * 5, [0] * 5, 100, 3) == ([0, 1, 2], 6)
    # running requests project I + g + 1
    assert O.pack_batch([1, 0], [5, 5], [0, 10], 100, 64) == ([1, 0], 16 + 6)
    # cut vs skip: the big request blocks the cut scan, the skip scan passes it
    # (request 1 is a running one whose KV grew to I + g = 35)
    I, g = [3, 5, 4], [0, 30, 0]
    assert O.pack_batch([0, 1, 2], I, g, 20, 64, "cut") == ([0], 4)
    assert O.pack_batch([0, 1, 2], I, g, 20, 64, "skip") == ([0, 2], 9)
    # a request with I + 1 > K can never run
    with pytest.raises(ValueError, match="cannot fit"):
        O.pack_batch([0], [20], [0], 20, 64)
    assert O.pack_batch([], [], [], 8192, 64) == ([], 0)

"""Trace generator and JSON Lines format:
the SPEC's own examples and invariants, on the host."""

import json
import warnings

import numpy as np
import pytest

from paper_2603_07917_b200.trace import (ClusterSpec, LengthLaw, Request, TraceError,
                                         WorkloadConfig, generate_trace, load_trace, save_trace)


def _cfg(lam=1.0, n=3, seed=7, law=LengthLaw("lognormal", (5.0, 1.0)), o_max=2048, nclusters=3):
    cl = tuple(ClusterSpec(tuple(range(100 * c, 100 * c + 20)), 8, law) for c in range(nclusters))
    return WorkloadConfig(lam=lam, n_requests=n, clusters=cl, seed=seed, o_max=o_max)


def test_generate_deterministic(tmp_path):
    # SPEC.md:51 "cfg{lambda=1, n=3, seed=7} run twice -> byte-identical traces"
    a, b = tmp_path / "a.jsonl", tmp_path / "b.jsonl"
    save_trace(generate_trace(_cfg()), str(a))
    save_trace(generate_trace(_cfg()), str(b))
    assert a.read_bytes() == b.read_bytes()
    t = generate_trace(_cfg(n=50))
    assert [r.id for r in t] == list(range(50))
    assert all(t[i].arrival_time <= t[i + 1].arrival_time for i in range(49))
    assert all(r.input_len == len(r.prompt_tokens) == 28 for r in t)


def test_generate_poisson_mean_gap():
    # SPEC.md:52 "cfg{lambda=4, n=100000, seed=1} -> mean gap within 2% of 0.25 s"
    t = generate_trace(_cfg(lam=4.0, n=100_000, seed=1, nclusters=1))
    gap = t[-1].arrival_time / len(t)
    assert abs(gap - 0.25) / 0.25 < 0.02


def test_generate_degenerate_geometric():
    # SPEC.md:53 "geometric(p=1.0) length law -> every true_output_len = 1"
    t = generate_trace(_cfg(n=200, law=LengthLaw("geometric", (1.0,))))
    assert {r.true_output_len for r in t} == {1}


def test_length_histogram_converges():
    # single-cluster trace, TV distance < 0.05 at n = 50,000
    p, o_max = 0.01, 2048
    t = generate_trace(_cfg(n=50_000, seed=3, law=LengthLaw("geometric", (p,)), nclusters=1))
    o = np.array([r.true_output_len for r in t])
    assert o.min() >= 1 and o.max() <= o_max
    v = np.arange(1, o_max + 1)
    pmf = (1 - p) ** (v - 1) * p
    pmf /= pmf.sum()
    emp = np.bincount(o, minlength=o_max + 1)[1:] / o.size
    assert 0.5 * np.abs(emp - pmf).sum() < 0.05


def test_truncation_clamps():
    t = generate_trace(_cfg(n=100, law=LengthLaw("bimodal", (5000.0, 0.5, 3000.0)), o_max=100))
    assert {r.true_output_len for r in t} == {100}


def test_roundtrip_and_empty(tmp_path):
    # SPEC.md:63-65
    t = generate_trace(_cfg(n=3))
    f = tmp_path / "t.jsonl"
    save_trace(t, str(f))
    assert load_trace(str(f)) == t
    e = tmp_path / "e.jsonl"
    e.write_text("")
    assert load_trace(str(e)) == []


def test_malformed_rejected_with_line(tmp_path):
    # SPEC.md:64 "input_len != prompt length -> rejection at the offending line"
    f = tmp_path / "bad.jsonl"
    good = {"id": 0, "arrival_time": 0.5, "prompt_tokens": [1, 2], "input_len": 2,
            "true_output_len": 3}
    bad = dict(good, id=1, input_len=5)
    f.write_text(json.dumps(good) + "\n" + json.dumps(bad) + "\n")
    with pytest.raises(TraceError, match=r"bad.jsonl:2:"):
        load_trace(str(f))
    f.write_text(json.dumps(good) + "\n{not json\n")
    with pytest.raises(TraceError, match=r":2:"):
        load_trace(str(f))
    f.write_text(json.dumps({k: v for k, v in good.items() if k != "true_output_len"}) + "\n")
    with pytest.raises(TraceError, match=r":1:.*missing"):
        load_trace(str(f))


def test_unsorted_resorted_with_warning(tmp_path):
    # stable sort by arrival_time, tie-break by id, with a warning
    recs = [Request(2, 1.0, (1,), 1, 1), Request(0, 2.0, (1,), 1, 1), Request(1, 1.0, (1,), 1, 1)]
    f = tmp_path / "u.jsonl"
    save_trace(recs, str(f))
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        out = load_trace(str(f))
    assert [r.id for r in out] == [1, 2, 0]
    assert any("re-sorted" in str(x.message) for x in w)


def test_config_errors_name_the_field():
    with pytest.raises(TraceError, match="lam"):
        generate_trace(WorkloadConfig(lam=0.0, n_requests=1, clusters=_cfg().clusters))
    with pytest.raises(TraceError, match="n_requests"):
        generate_trace(WorkloadConfig(lam=1.0, n_requests=0, clusters=_cfg().clusters))
    with pytest.raises(TraceError, match="length_law"):
        LengthLaw("geometric", (1.5,))

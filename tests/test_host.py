"""Host-side logic of the drop-in (no GPU): the DiscreteDistribution
container, the scalar cost API, configs, priorities and the no-fallback rule."""

import numpy as np
import pytest
import torch

from paper_2603_07917_b200 import _lib
from paper_2603_07917_b200.cost import (OutputOnly, ResourceBound, WeightedSum, CostUnits, cost,
                                        parse_cost_kind, remaining_cost)
from paper_2603_07917_b200.distribution import (DiscreteDistribution, DistributionError,
                                                total_variation)
from paper_2603_07917_b200.gittins import GittinsConfig, ServiceProgress, refresh_due
from paper_2603_07917_b200.policies import Priority
from paper_2603_07917_b200.scheduler import RoundConfig


def test_distribution_contract():
    d = DiscreteDistribution([3, 1, 2, 1], [0.25, 0.25, 0.25, 0.25])
    assert list(d.support) == [1, 2, 3] and list(d.masses) == [0.5, 0.25, 0.25]
    d = DiscreteDistribution([1, 2, 3], [0.5, 0.0, 0.5])
    assert list(d.support) == [1, 3]
    for bad in ([], [1.0, np.inf]):
        with pytest.raises(DistributionError):
            DiscreteDistribution(bad, [1.0] * len(bad))
    with pytest.raises(DistributionError):
        DiscreteDistribution([1, 2], [0.5, 0.6])
    with pytest.raises(DistributionError):
        DiscreteDistribution([1, 2], [-0.5, 1.5])
    with pytest.raises(DistributionError):
        DiscreteDistribution([1], [1.0, 0.0])
    assert issubclass(DistributionError, ValueError)
    e = DiscreteDistribution.from_samples([1, 9, 9, 1])
    assert list(e.support) == [1, 9] and list(e.masses) == [0.5, 0.5]
    assert e.mean() == 5.0 and e.mass_at(9) == 0.5 and e.mass_at(4) == 0.0
    assert total_variation(e, e) == 0.0
    assert total_variation(DiscreteDistribution.from_pairs({1: .5, 9: .5}),
                           DiscreteDistribution.point(1)) == 0.5
    u = DiscreteDistribution.uniform_integers(1, 4)
    assert len(u) == 4 and abs(u.masses.sum() - 1) < 1e-12
    with pytest.raises(DistributionError):
        e.map_support(lambda x: -x)


def test_cost_scalar_api():
    assert cost(ResourceBound(), 100, 200) == 40000
    assert cost(OutputOnly(), 5000, 10) == 10
    assert cost(WeightedSum(1, 2), 100, 50) == 200
    assert remaining_cost(ResourceBound(), 100, 200, 100) == 25000
    assert remaining_cost(ResourceBound(), 100, 200, 200) == 0
    with pytest.raises(ValueError):
        cost(ResourceBound(), 0, 5)
    with pytest.raises(ValueError):
        cost(ResourceBound(), 5, -1)
    with pytest.raises(ValueError):
        remaining_cost(ResourceBound(), 1, 5, 6)
    with pytest.raises(TypeError):
        cost(object(), 1, 1)
    with pytest.raises(ValueError):
        WeightedSum(0, 1)
    with pytest.raises(ValueError):
        CostUnits(0, 1)
    assert parse_cost_kind("weighted-sum", w_in=2.0) == WeightedSum(2.0, 2.0)
    with pytest.raises(ValueError):
        parse_cost_kind("nope")
    rng = np.random.default_rng(0)
    for I, O, o in zip(rng.integers(1, 4097, 1000), rng.integers(0, 2049, 1000),
                       rng.integers(0, 2049, 1000)):
        o = min(o, O)
        assert remaining_cost(ResourceBound(), I, O, o) + cost(ResourceBound(), I, o) == \
            cost(ResourceBound(), I, O)


def test_refresh_and_progress():
    p = ServiceProgress(199, cost(ResourceBound(), 10, 199), 0)
    assert refresh_due(p, 200)
    p = ServiceProgress(200, 0.0, 1)
    assert not refresh_due(p, 399)
    p = ServiceProgress(150, 0.0, 0)
    assert refresh_due(p, 650)
    with pytest.raises(ValueError):
        refresh_due(p, 100)
    with pytest.raises(ValueError):
        GittinsConfig(bucket_size_tokens=0)
    nxt = ServiceProgress.start().advance(ResourceBound(), 100, 450)
    assert nxt.current_bucket == 2 and nxt.attained_cost == cost(ResourceBound(), 100, 450)


def test_configs_and_priority_order():
    with pytest.raises(ValueError):
        RoundConfig(k=0)
    with pytest.raises(ValueError):
        RoundConfig(max_len=2048, nbins=100)
    a = Priority(2.0, (1.0, 5))
    b = Priority(2.0, (1.0, 6))
    c = Priority(1.0, (9.0, 9))
    assert sorted([a, b, c]) == [c, a, b]


def test_product_path_has_no_cpu_fallback():
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_07917_b200 import _kernels
    with pytest.raises(_lib.CudaExtensionMissing):
        _kernels.gittins_min(np.array([1.0]), np.array([1.0]))
    with pytest.raises(_lib.CudaExtensionMissing):
        from paper_2603_07917_b200.history import HistoryWindow
        HistoryWindow(16, 384)


def test_product_package_never_imports_oracle():
    import pathlib
    pkg = pathlib.Path(_lib.__file__).parent
    for f in pkg.glob("*.py"):
        assert "oracle" not in f.read_text().replace("oracle/", ""), f


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the driver's reference arm) runs on the host
    cores and prints one JSON line with the contract's keys."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True,
                       timeout=600, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "cpu_baseline", "e2e", "config"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["cores"] >= 1 and line["e2e"]["h2d_bytes_per_step"] == 0

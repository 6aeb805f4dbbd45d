"""Per-call latency of the reference-signature drop-ins against the
reference's numba/numpy calls (baseline/_ref), on this box.  One law / one
request per call, as a SPEC engine calls them."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")


def per_call_us(fn, n=2000):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    import torch

    from paper_2603_07917_b200 import _kernels as K
    from paper_2603_07917_b200 import cost as Cst
    from paper_2603_07917_b200.distribution import DiscreteDistribution
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.predictor import Request, SemanticHistory, predict
    from paper_2603_07917_b200.synthetic import make_bank_device
    torch.cuda.init()
    rng = np.random.default_rng(0)
    sup = np.sort(rng.choice(np.arange(1, 5_000_000), 512, replace=False)).astype(np.float64)
    mas = rng.random(512)
    mas /= mas.sum()
    out = {"box_cores": os.cpu_count()}
    out["ours_gittins_min_512pt_us"] = per_call_us(lambda: K.gittins_min(sup, mas))
    d = DiscreteDistribution(sup[:64], mas[:64] / mas[:64].sum())
    rb = Cst.ResourceBound()
    out["ours_cost_distribution_64pt_us"] = per_call_us(lambda: Cst.cost_distribution(rb, 100, d))
    try:
        from servesim import _kernels as RK
        from servesim import cost as RC
        from servesim.distribution import DiscreteDistribution as RD
        RK.warmup()
        out["ref_gittins_min_512pt_us"] = per_call_us(lambda: RK.gittins_min(sup, mas))
        rd = RD(sup[:64], mas[:64] / mas[:64].sum())
        out["ref_cost_distribution_64pt_us"] = per_call_us(lambda: RC.cost_distribution(RC.ResourceBound(), 100, rd))
    except Exception as e:  # noqa: BLE001
        out["ref_unavailable"] = repr(e)
    emb, lens, _ = make_bank_device(100_000, 384, 1000, 0)
    w = HistoryWindow(100_000, 384)
    w.push(emb, lens)
    req = Request(0, rng.integers(0, 50000, 300))
    kind = SemanticHistory()
    predict(kind, req, w)
    out["ours_predict_100k_window_us"] = per_call_us(lambda: predict(kind, req, w), n=300)
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in out.items()}))


if __name__ == "__main__":
    main()

"""One small scheduling round of every stage-1 kernel instantiation plus the
merge/finish/rank kernels, for compute-sanitizer (racecheck / memcheck /
synccheck).  Kept small: the sanitizers replay every access.

    compute-sanitizer --tool racecheck python scripts/sanitize_round.py
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import sagesched_oracle as O  # noqa: E402
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler  # noqa: E402


def main():
    _lib.load()
    n = 6000
    emb, lens, _, _ = O.make_bank(n + 300, 384, 30, 3)
    w = HistoryWindow(n, 384)
    w.push(emb[:n], lens[:n])
    I = np.random.default_rng(1).integers(1, 4097, 300).astype(np.int32)
    ok = True
    # nq = 300: k_topk_ts (theta 0.8: locked shared heaps; theta -1: the
    # pure top-k cascade -- threshold pass, then the SHARE instantiation for
    # unresolved tiles, forced by random queries) + k_merge_finish_w + rank;
    # nq = 64: k_topk_tc
    rq = np.random.default_rng(2).integers(-60, 61, (300, 384)).astype(np.int8)
    for nq, theta, rand in ((300, 0.8, False), (300, -1.0, False), (300, -1.0, True), (64, 0.8, False),
                            (64, -1.0, False)):
        q = rq[:nq] if rand else emb[n:n + nq]
        qi = O.inv_norm(q)
        cfg = RoundConfig(k=32, theta=theta, min_matches=20, nbins=64)
        perm, G, _ = SageScheduler(w, cfg).schedule_round(
            torch.as_tensor(q, device="cuda"), torch.as_tensor(qi, device="cuda"),
            torch.as_tensor(I[:nq], device="cuda"), torch.arange(nq, device="cuda"))
        torch.cuda.synchronize()
        keys = O.scores(q, qi, emb[:n], O.inv_norm(emb[:n]))
        ref = O.predict_round(keys, np.arange(n), lens[:n], I[:nq], 32, theta, 20, 2048, 64,
                              window_lens=lens[:n])
        good = np.array_equal(G.cpu().numpy(), np.array([r["G"] for r in ref]))
        print(f"nq={nq} theta={theta}{' random queries' if rand else ''}: {'ok' if good else 'MISMATCH'}")
        ok &= good
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()

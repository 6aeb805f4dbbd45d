"""Parity check of the stage-1 kernel the library picks under the current
SS_TC_* environment (run in a subprocess by tests/test_gpu_variants.py, since
the library reads those switches once per process)."""

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import sagesched_oracle as O  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402


def main():
    n, nq = int(sys.argv[1]), int(sys.argv[2])
    for theta, k in ((0.8, 64), (0.3, 64), (-1.0, 32)):
        emb, lens, _, _ = O.make_bank(n + nq, 384, 64, 5)
        w = HistoryWindow(n, 384)
        w.push(emb[:n], lens[:n])
        q = emb[n:]
        qi = O.inv_norm(q)
        keys = O.scores(q, qi, emb[:n], O.inv_norm(emb[:n]))
        seq = np.arange(n)
        comp, ln = w.topk(q, qi, k, theta, "tcgen05")
        key, gseq, _ = w.decode(comp)
        key, gseq, ln = key.cpu().numpy(), gseq.cpu().numpy(), ln.cpu().numpy()
        for i in range(nq):
            sel = O.select_topk(keys[i], seq, k, theta)
            m = sel.size
            assert np.array_equal(gseq[i, :m], seq[sel]), (theta, i)
            assert np.array_equal(key[i, :m], keys[i, sel]), (theta, i)
            assert np.array_equal(ln[i, :m], lens[sel]), (theta, i)
            assert np.all(gseq[i, m:] == -1), (theta, i)
    print("ok")


if __name__ == "__main__":
    main()

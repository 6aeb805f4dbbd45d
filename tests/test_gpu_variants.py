"""The opt-in stage-1 kernels (selected by SS_TC_* switches the library reads
once per process) stay bit-exact: each runs in its own subprocess."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("env", [{"SS_TC_PAIR": "1"}, {"SS_TC_TSN": "256"}, {"SS_TC_TSN": "192"},
                                 {"SS_TC_TSN": "224"},
                                 {"SS_TC_TS": "0"}, {"SS_TC_TS": "0", "SS_TC_GTHR": "1"},
                                 {"SS_TC_SHARE": "0"},
                                 {"SS_TC_TS": "0", "SS_TC_CG": "2"}])
def test_topk_variant_bit_exact(cuda, env):
    _check_variant(env, 30000, 600)


@pytest.mark.parametrize("env,n,nq", [({"SS_TC_MC": "1"}, 30000, 1000),
                                      ({"SS_TC_MC": "1"}, 100_003, 256),
                                      ({"SS_TC_MC": "1", "SS_TC_TSN": "256"}, 30000, 512),
                                      ({"SS_TC_MC": "1", "SS_TC_TSN": "224"}, 30000, 512),
                                      ({"SS_TC_MC": "1", "SS_TC_TSN": "512"}, 30000, 1000),
                                      ({"SS_TC_TSN": "512"}, 30000, 600)])
def test_topk_multicast_pairs_bit_exact(cuda, env, n, nq):
    """2-CTA clusters sharing each bank tile by TMA multicast (even query-tile
    counts; ragged last tile and last query tile included)."""
    _check_variant(env, n, nq)


def _check_variant(env, n, nq):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "check_topk_variant.py"),
                        str(n), str(nq)], env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]

"""c4 on N GPUs from components measured on ONE B200 (a projection, not a
multi-GPU measurement: one GPU is reachable from this build).

The single-owner round at world N is
    broadcast(queue) -> every rank: local fused top-k of the 8192 queries
    against its 16M/N-row shard -> all-gather of k candidates per query ->
    owner: merge N x k per query, histogram -> cost -> Gittins, rank.
Here the 16M-row bank is built once, cut into N contiguous shards exactly as
``ShardPlan`` places them (global slots [r L, (r+1) L), composites carry the
global ring rank), and on this one GPU:
  * every shard's local stage (``HistoryWindow.topk``: the TS kernel + its
    slice merge) is timed with CUDA events, one shard after another;
  * the owner's stages (``ss_merge_topk`` of the N lists, ``ss_finish``,
    ``ss_rank``) are timed on the stacked shard outputs;
  * the merged lists are checked bit-for-bit against the unsharded 16M-row
    round's lists (same composites, same lengths) and G / order equality.
The two collectives are not run; they are charged from the profiling
recipe's measured NVLink figures (B200_PROFILING.md: 770 GB/s peer copy per
direction, 725 GB/s all-reduce bus bandwidth at 1 GiB) plus a fixed 15 us
launch/latency each -- stated in the output.
Projected round(N) = max over shards of the local stage + broadcast +
all-gather + owner stages.  Writes one JSON object to stdout.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import rank  # noqa: E402
from paper_2603_07917_b200.sharded import ShardPlan  # noqa: E402
from paper_2603_07917_b200.synthetic import make_bank_device, make_queries  # noqa: E402

DIM, K, NBINS, MAX_LEN, THETA, MIN_MATCHES, N_CLUSTERS, SEED = 384, 64, 128, 2048, 0.8, 20, 4096, 0
NVLINK_GBS, LAT_US = 770.0, 15.0


def ev_ms(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def owner_stages(comp_x, len_x, nlists, nq, I, fb, ids):
    comp = torch.empty((nq, K), dtype=torch.int64, device="cuda")
    ln = torch.empty((nq, K), dtype=torch.int32, device="cuda")
    out = dict(npts=torch.zeros(nq, dtype=torch.int32, device="cuda"),
               pbin=torch.zeros((nq, NBINS), dtype=torch.int32, device="cuda"),
               pcnt=torch.zeros((nq, NBINS), dtype=torch.int32, device="cuda"),
               pD=torch.zeros((nq, NBINS), dtype=torch.int64, device="cuda"),
               used_fb=torch.zeros(nq, dtype=torch.uint8, device="cuda"),
               G=torch.empty(nq, dtype=torch.float64, device="cuda"))
    perm = torch.empty(nq, dtype=torch.int64, device="cuda")
    ws = torch.empty(int(_lib.lib().ss_rank_workspace_bytes(nq)), dtype=torch.uint8, device="cuda")
    P = _lib.ptr

    def go():
        if nlists > 1:
            _lib.call("ss_merge_topk", P(comp_x), P(len_x), nlists, nq, K, P(comp), P(ln),
                      _lib.stream_ptr())
            c, l_ = comp, ln
        else:
            c, l_ = comp_x, len_x
        _lib.call("ss_finish", P(c), P(l_), nq, K, MIN_MATCHES, MAX_LEN, NBINS, P(I), P(fb[0]),
                  P(fb[1]), P(fb[2]), NBINS, P(out["npts"]), P(out["pbin"]), P(out["pcnt"]),
                  P(out["pD"]), None, P(out["used_fb"]), P(out["G"]), _lib.stream_ptr())
        rank(out["G"], ids, perm, ws)
    return go, (comp if nlists > 1 else comp_x), (ln if nlists > 1 else len_x), out, perm


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=1 << 24)
    ap.add_argument("--nq", type=int, default=8192)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    _lib.load()
    n, nq = a.rows, a.nq
    emb, lens, _ = make_bank_device(n, DIM, N_CLUSTERS, SEED)
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))

    # the unsharded reference round on this GPU (16M-row window)
    full = HistoryWindow(n, DIM)
    full.push(emb, lens)
    fb_full = full.fallback_hist(MAX_LEN, NBINS)
    t_full = ev_ms(lambda: full.topk(dq, dqi, K, THETA), a.reps)
    c_full, l_full = full.topk(dq, dqi, K, THETA)
    go1, _, _, out1, perm1 = owner_stages(c_full, l_full, 1, nq, dI, fb_full, dids)
    t_own1 = ev_ms(go1, a.reps)
    go1()
    torch.cuda.synchronize()
    G1, p1 = out1["G"].clone(), perm1.clone()
    del full
    torch.cuda.empty_cache()

    res = {"what": "c4 single-owner round on N GPUs projected from components measured on one "
                   "B200 (not a multi-GPU measurement)",
           "rows": n, "nq": nq, "k": K, "theta": THETA,
           "one_gpu": {"local_topk_ms": round(t_full, 3), "owner_ms": round(t_own1, 3),
                       "round_ms": round(t_full + t_own1, 3)},
           "collective_model": f"{NVLINK_GBS} GB/s per direction (B200_PROFILING.md peer copy) + "
                               f"{LAT_US} us per collective", "worlds": []}
    for world in [int(w) for w in a.worlds.split(",")]:
        L = n // world
        comps, lns, times = [], [], []
        fb = torch.zeros((3, NBINS), dtype=torch.int64, device="cuda")
        for r in range(world):
            plan = ShardPlan(n, world, r)  # the sharded round's own placement
            w = HistoryWindow(plan.local_capacity, DIM, global_capacity=n, slot_offset=plan.slot_offset)
            idx, seq, slot = (torch.as_tensor(x, device="cuda") for x in plan.route(0, n))
            w.write(emb[idx], lens[idx], seq, slot)
            w.set_head(n)
            del idx, seq, slot
            fb += w.fallback_hist(MAX_LEN, NBINS)
            times.append(ev_ms(lambda: w.topk(dq, dqi, K, THETA), a.reps))
            c, l_ = w.topk(dq, dqi, K, THETA)
            comps.append(c)
            lns.append(l_)
            del w
            torch.cuda.empty_cache()
        comp_x, len_x = torch.stack(comps).contiguous(), torch.stack(lns).contiguous()
        go, comp, ln, out, perm = owner_stages(comp_x, len_x, world, nq, dI, fb, dids)
        t_own = ev_ms(go, a.reps)
        go()
        torch.cuda.synchronize()
        exact = bool(torch.equal(comp, c_full) and torch.equal(ln, l_full) and torch.equal(fb, fb_full)
                     and torch.equal(out["G"], G1) and torch.equal(perm, p1))
        bcast_b = nq * (DIM + 4)
        gather_b = (world - 1) * nq * K * 12  # the owner receives every other rank's lists
        t_coll = (bcast_b + gather_b) / (NVLINK_GBS * 1e9) * 1e3 + 2 * LAT_US / 1e3
        t_round = max(times) + t_coll + t_own
        res["worlds"].append({
            "n_gpus": world, "shard_rows": L, "local_topk_ms_per_shard": [round(t, 3) for t in times],
            "owner_merge_finish_rank_ms": round(t_own, 3), "collectives_ms_modelled": round(t_coll, 3),
            "projected_round_ms": round(t_round, 3),
            "projected_requests_per_s": round(nq / (t_round / 1e3), 1),
            "bit_identical_to_one_gpu_round": exact})
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()

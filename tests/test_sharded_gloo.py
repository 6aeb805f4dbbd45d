"""Multi-GPU host logic on CPU: shard routing of the global FIFO ring and the
query all-gather / candidate all-to-all / histogram all-reduce exchange of
paper_2603_07917_b200.sharded, run with world_size 2 over gloo.  The local
top-k and the merge are the CPU oracle here (the kernels need a GPU); the
result must equal the single-bank oracle top-k bit for bit."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import sagesched_oracle as O
from paper_2603_07917_b200.sharded import (ShardPlan, allreduce_hist, exchange_candidates,
                                           gather_queries)


def f32_order(x):
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    return np.where(b & 0x80000000, (~b) & 0xFFFFFFFF, b | 0x80000000)


def composites(keys_row, seq, sel, head, cap):
    rel = (np.asarray(seq)[sel] % cap - head % cap) % cap
    return (f32_order(keys_row[sel]) << np.uint64(32)) | rel.astype(np.uint64)


def test_shard_plan_matches_ring_model():
    rng = np.random.default_rng(0)
    for world in (1, 2, 4, 8):
        cap = 64 * world
        ring = {}
        head = 0
        for _ in range(20):
            n = int(rng.integers(1, 3 * cap))
            got = {}
            for r in range(world):
                p = ShardPlan(cap, world, r)
                idx, seq, slot = p.route(head, n)
                for i, s, l in zip(idx, seq, slot):
                    g = p.slot_offset + l
                    assert g not in got
                    got[g] = s
                    assert 0 <= l < p.local_capacity
            for i in range(n):
                ring[(head + i) % cap] = head + i
            head += n
            expect = {g: s for g, s in ring.items() if s >= head - n}  # written this push
            assert got == expect
    with pytest.raises(ValueError):
        ShardPlan(10, 3, 0)


def _worker(rank, world, port, result_q):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    try:
        dim, n_total, nq, k, theta = 128, 4000, 24, 16, -1.0
        emb, lens, _, _ = O.make_bank(n_total + nq * world, dim, 30, seed=5)
        bank_e, bank_l = emb[:n_total], lens[:n_total]
        cap = n_total
        head = n_total
        seq = np.arange(n_total)
        plan = ShardPlan(cap, world, rank)
        lo, hi = plan.slot_offset, plan.slot_offset + plan.local_capacity
        # this rank's own queue
        q = emb[n_total + rank * nq: n_total + (rank + 1) * nq]
        qi = O.inv_norm(q)
        q_all, qi_all = gather_queries(torch.as_tensor(q), torch.as_tensor(qi))
        q_all, qi_all = q_all.numpy(), qi_all.numpy()
        # local top-k of ALL queries against this shard (oracle stand-in for ss_topk)
        keys = O.scores(q_all, qi_all, bank_e[lo:hi], O.inv_norm(bank_e[lo:hi]))
        comp = np.zeros((world * nq, k), np.uint64)
        ln = np.zeros((world * nq, k), np.int32)
        for i in range(world * nq):
            sel = O.select_topk(keys[i], seq[lo:hi], k, theta)
            comp[i, :sel.size] = composites(keys[i], seq[lo:hi], sel, head, cap)
            ln[i, :sel.size] = bank_l[lo:hi][sel]
        cx, lx = exchange_candidates(torch.as_tensor(comp.view(np.int64)), torch.as_tensor(ln))
        cx = cx.numpy().view(np.uint64)
        lx = lx.numpy()
        # merge (oracle stand-in for ss_merge_topk) and compare with the global oracle
        gkeys = O.scores(q, qi, bank_e, O.inv_norm(bank_e))
        ok = True
        for i in range(nq):
            allc = cx[:, i, :].reshape(-1)
            alll = lx[:, i, :].reshape(-1)
            order = sorted(np.flatnonzero(allc), key=lambda j: -int(allc[j]))[:k]
            sel = O.select_topk(gkeys[i], seq, k, theta)
            ref = composites(gkeys[i], seq, sel, head, cap)
            ok &= np.array_equal(allc[order], ref)
            ok &= np.array_equal(alll[order], bank_l[sel])
        # fallback histogram: per-shard exact sums
        h = torch.as_tensor(np.stack(O.bin_hist(bank_l[lo:hi], 2048, 64)))
        allreduce_hist(h)
        ok &= np.array_equal(h.numpy(), np.stack(O.bin_hist(bank_l, 2048, 64)))
        result_q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_equals_global_topk():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    results = dict(q.get(timeout=10) for _ in range(2))
    assert results == {0: True, 1: True}

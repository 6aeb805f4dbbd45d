"""Worker of test_gpu_parity.test_sharded_p2p_two_ranks_one_gpu (not a test module).

Two ranks share cuda:0 (gloo carries the collectives: NCCL refuses two ranks
on one device).  Each rank holds half of the ring.  Mode "per-rank": each
rank has its own queue; mode "owner" (argv[1]): rank 1 owns the whole queue;
both use the fused P2P merge + exchange, whose stores cross the process
boundary through the IPC mapping.  Mode "owner-coll": rank 1 owns the whole
queue and the round uses the collective exchange (broadcast of the queue,
all-gather of k candidates per query, all-reduce of the window histogram --
NCCL on a real node, gloo on CUDA tensors here).  Every queue owner checks its
Gittins indices and order against the single-GPU round over the whole bank.
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import sagesched_oracle as O  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler  # noqa: E402
from paper_2603_07917_b200.sharded import ShardedHistory, ShardedScheduler  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    n, dim, nq = 12_000, 384, 96
    emb, lens, _, _ = O.make_bank(n + world * nq, dim, 40, 3)
    cfg = RoundConfig(k=32, theta=0.7, nbins=64)
    sh = ShardedHistory(n, dim)
    sh.push(torch.as_tensor(emb[:n], device="cuda"), torch.as_tensor(lens[:n], device="cuda"))
    lo = n + rank * nq
    q = torch.as_tensor(emb[lo:lo + nq], device="cuda")
    qi = torch.as_tensor(O.inv_norm(emb[lo:lo + nq]), device="cuda")
    I = torch.as_tensor(np.random.default_rng(rank).integers(1, 4097, nq).astype(np.int32),
                        device="cuda")
    ids = torch.arange(rank * nq, (rank + 1) * nq, device="cuda")
    mode = sys.argv[1] if len(sys.argv) > 1 else "per-rank"
    if mode in ("owner", "owner-coll"):  # rank 1 owns the whole queue (both halves)
        q = torch.as_tensor(emb[n:n + world * nq], device="cuda")
        qi = torch.as_tensor(O.inv_norm(emb[n:n + world * nq]), device="cuda")
        I = torch.as_tensor(np.random.default_rng(7).integers(1, 4097, world * nq).astype(np.int32),
                            device="cuda")
        ids = torch.arange(world * nq, device="cuda")
        ss = ShardedScheduler(sh, cfg, exchange="p2p" if mode == "owner" else "nccl", owner=1)
    else:
        ss = ShardedScheduler(sh, cfg, exchange="p2p", owner=None)
    mine = mode == "per-rank" or rank == 1
    for _ in range(3):  # receive buffers reused across rounds
        if mine:
            p1, G1, _ = ss.schedule_round(q, qi, I, ids)
        else:
            assert ss.schedule_round(None, None, nq=world * nq) is None
        torch.cuda.synchronize()
        dist.barrier()
    ok = True
    if mine:
        delivered = True
        if mode != "owner-coll":
            # the peer's shard really delivered rows into this rank's receive buffer
            recv = ss.peer.buffers(q.shape[0])["recv_c"]
            delivered = bool(recv[1 - rank].ne(0).any()) and bool(recv[rank].ne(0).any())
        w = HistoryWindow(n, dim)
        w.push(emb[:n], lens[:n])
        p0, G0, _ = SageScheduler(w, cfg).schedule_round(q, qi, I, ids)
        ok = delivered and torch.equal(G1, G0) and torch.equal(p1, p0)
    if ss.peer is not None:
        ss.peer.close()
    dist.barrier()
    dist.destroy_process_group()
    if not ok:
        print(f"rank {rank}: sharded round ({mode}) differs from the single-GPU round", file=sys.stderr)
        sys.exit(1)


if __name__ == "__main__":
    main()

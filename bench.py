"""Benchmark of the SageSched per-round scheduling hot path on B200.

One step = one scheduling round over one batch of synthetic pending requests:
predict (1M x 384 int8 history bank -> top-64 -> 128-bin length histogram)
-> cost (O^2/2 + I*O) -> Gittins index -> rank.  Workload = BASELINE.json
configs[1] ("1M-entry bank, 1024 pending prompts per round, k=64, 128 bins").

  value  requests scheduled / s with inputs resident in HBM (CUDA-graph replay
         of the fused round, CUDA events, max over ranks)
  e2e    same metric through the plugin call from pinned HOST buffers
         (ss_schedule_round_host: H2D + round + D2H inside the timed region)

``--impl reference`` times the reference's CPU implementation of the path
(servesim from baseline/_ref where the code exists, the oracle restatement of
the SPEC-only pieces) on a bounded sample, on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_BANK, DIM, NQ, K, NBINS, MAX_LEN = 1 << 20, 384, 1024, 64, 128, 2048
THETA, MIN_MATCHES, N_CLUSTERS = 0.8, 20, 4096
SEED = 0
WORKLOAD = "c2: 1M-entry x 384-d int8 history bank, 1024 pending prompts/round, k=64, 128 bins"


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "_fallback": True}


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self):
        return time.time()

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self, t0, t1):
        rows = [l for (t, l) in self.lines if t0 - 0.06 <= t <= t1 + 0.06] or \
               [l for (_, l) in self.lines[-3:]]
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            p = [x.strip() for x in r.split(",")]
            if len(p) < 6:
                continue
            try:
                sm.append(float(p[0]))
                mx = float(p[1])
            except ValueError:
                continue
            for n, v in zip(names, p[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ our arm -----
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_07917_b200 import _build, _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    # SS_BENCH_SHARDED=1 runs the sharded (multi-GPU) round even at N = 1,
    # under torchrun, so its code path can be exercised on one GPU
    sharded = world > 1 or os.environ.get("SS_BENCH_SHARDED") == "1"
    if sharded:
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    if _build.is_stale() and rank == 0:
        _build.build()
    if sharded:
        dist.barrier()
    _lib.load()

    if sharded:
        return run_sharded(args, world, rank, local)
    emb, lens, _ = make_bank_device(N_BANK, DIM, N_CLUSTERS, SEED)
    win = HistoryWindow(N_BANK, DIM)
    win.push(emb, lens)
    del emb, lens
    q, qi, I, ids = make_queries(NQ, DIM, N_CLUSTERS, SEED, qseed=1000 + rank)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS,
                      algo=args.algo)
    sched = SageScheduler(win, cfg)

    # launches per round (counted on an eager round)
    c0 = _lib.launch_count()
    sched.schedule_round(dq, dqi, dI, dids)
    torch.cuda.synchronize()
    per_round = _lib.launch_count() - c0

    graph, out = sched.capture_round(dq, dqi, dI, dids)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(local)
    with sampler:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            graph.replay()
        ev1.record()
        torch.cuda.synchronize()
        t1 = time.time()
        if world > 1:
            dist.barrier()
        ms = ev0.elapsed_time(ev1)
        clocks = sampler.summary(t0, t1)

        # dominant kernel alone (similarity + fused top-k), same stream, CUDA events
        algo_used, kern_ms, n_slices = time_topk_kernel(sched, dq, dqi, args)

        # e2e: plugin call from pinned host buffers
        e2e_ms, h2d, d2h = time_e2e(sched, q, qi, I, ids, args)

    # max over ranks
    vals = torch.tensor([ms, e2e_ms, kern_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, kern_ms = vals.tolist()

    if rank == 0:
        pk = peaks()
        req = NQ * world
        value = req * args.steps / (ms / 1e3)
        kern_s = kern_ms / 1e3
        if algo_used == "tcgen05":
            ops = 2.0 * NQ * N_BANK * DIM
            achieved = ops / kern_s / 1e12
            peak = 2.0 * pk["bf16_tflops"]
            roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                    "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                    "peak_source": "int8 dense = 2 x measured bf16 burst (MEASURED_PEAKS.json)"}
        else:
            byts = N_BANK * DIM + N_BANK * 4.0 + NQ * DIM
            achieved = byts / kern_s / 1e9
            peak = pk["hbm_gbs"]
            roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4),
                    "peak_source": "measured copy bandwidth (MEASURED_PEAKS.json)"}
        roof["kernel"] = topk_kernel_name(algo_used, NQ)
        roof["kernel_ms"] = round(kern_ms, 4)
        roof["kernel_share_of_step"] = round(kern_ms / (ms / args.steps), 3)
        roof["traffic"] = ncu_traffic(roof["kernel"])
        line = {
            "metric": "requests scheduled/sec per round (predict+cost+Gittins+rank) vs a 1M-entry bank",
            "value": round(value, 1), "unit": "requests/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded clustered int8 embeddings, lognormal lengths)",
            "config": {"workload": WORKLOAD, "bank_rows": N_BANK, "dim": DIM, "nq": NQ, "k": K,
                       "nbins": NBINS, "theta": THETA, "min_matches": MIN_MATCHES,
                       "similarity": algo_used, "n_slices": n_slices,
                       "parallelism": f"replica x{world}" if world > 1 else "single GPU",
                       "l2": f"bank ({N_BANK * (DIM + 4) / 1e6:.0f} MB) > L2 (126 MB): every "
                             "round streams it from HBM"},
            "e2e": {"value": round(req * args.steps / (e2e_ms / 1e3), 1), "unit": "requests/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": round(e2e_ms / args.steps, 4)},
            "roofline": roof,
            "gpu_launches": int(per_round * args.steps),
            "clocks": clocks,
        }
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(budget_s=args.cpu_budget)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_sharded(args, world, rank, local):
    """N GPUs: the 1M-row bank is row-sharded (1M/N rows per GPU) and every
    rank owns a queue of 1024 pending prompts (weak scaling in requests:
    per-GPU similarity work stays 1024 x 1M).  Per round: query all-gather,
    local fused top-k of all N*1024 queries, candidate all-to-all, merge,
    histogram all-reduce, then cost/Gittins/rank of each rank's own queue."""
    import torch
    import torch.distributed as dist

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.scheduler import RoundConfig
    from paper_2603_07917_b200.sharded import ShardedHistory, ShardedScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    emb, lens, _ = make_bank_device(N_BANK, DIM, N_CLUSTERS, SEED)
    hist = ShardedHistory(N_BANK, DIM)
    hist.push(emb, lens)
    del emb, lens
    q, qi, I, ids = make_queries(NQ, DIM, N_CLUSTERS, SEED, qseed=1000 + rank)
    ids = ids + rank * NQ
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS,
                      algo=args.algo)
    # SS_SHARD_EXCHANGE=p2p: fused merge + exchange over IPC-mapped peer
    # buffers (ss_topk_scatter) instead of the candidate all_to_all
    exchange = os.environ.get("SS_SHARD_EXCHANGE", "nccl")
    sched = ShardedScheduler(hist, cfg, exchange=exchange)
    c0 = _lib.launch_count()
    sched.schedule_round(dq, dqi, dI, dids)
    torch.cuda.synchronize()
    per_round = _lib.launch_count() - c0
    # the whole sharded round (NCCL collectives included) as one CUDA graph;
    # eager rounds if this NCCL/driver combination cannot capture
    graph = None
    try:
        graph, _ = sched.capture_round(dq, dqi, dI, dids)
    except Exception as e:  # noqa: BLE001
        print(f"sharded round not captured ({type(e).__name__}: {e}); timing eager rounds",
              file=sys.stderr)
        graph = None
        torch.cuda.synchronize()

    def one_round():
        if graph is not None:
            graph.replay()
        else:
            sched.schedule_round(dq, dqi, dI, dids)

    for _ in range(args.warmup):
        one_round()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            one_round()
        e1.record()
        torch.cuda.synchronize()
        t1 = time.time()
        dist.barrier()
        ms = e0.elapsed_time(e1)
        clocks = sampler.summary(t0, t1)
        # e2e: pinned host queue in, order + indices out, every step
        hq, hqi, hI, hids = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
                             for x in (q, qi, I, ids))
        hG = torch.empty(NQ, dtype=torch.float64).pin_memory()
        hp = torch.empty(NQ, dtype=torch.int64).pin_memory()
        for _ in range(max(1, args.warmup)):  # first call captures the host round
            sched.schedule_round_host(hq, hqi, hI, hids, hG, hp)
        dist.barrier()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            sched.schedule_round_host(hq, hqi, hI, hids, hG, hp)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms = e0.elapsed_time(e1)
        # dominant kernel: the local similarity over all world*NQ queries
        q_all = torch.cat([dq] * world)
        qi_all = torch.cat([dqi] * world)
        algo_used, kern_ms, n_slices = time_topk_kernel(
            type("S", (), {"cfg": cfg, "window": hist.window})(), q_all, qi_all, args,
            nq=world * NQ)
    vals = torch.tensor([ms, e2e_ms, kern_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, kern_ms = vals.tolist()
    if rank == 0:
        pk = peaks()
        req = NQ * world
        ops = 2.0 * (world * NQ) * (N_BANK // world) * DIM
        achieved = ops / (kern_ms / 1e3) / 1e12
        peak = 2.0 * pk["bf16_tflops"]
        line = {
            "metric": "requests scheduled/sec per round (predict+cost+Gittins+rank) vs a 1M-entry bank",
            "value": round(req * args.steps / (ms / 1e3), 1), "unit": "requests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded clustered int8 embeddings, lognormal lengths)",
            "config": {"workload": WORKLOAD + f"; bank row-sharded over {world} GPUs, one "
                       f"1024-request queue per GPU", "bank_rows": N_BANK, "dim": DIM,
                       "nq_per_gpu": NQ, "k": K, "nbins": NBINS, "theta": THETA,
                       "similarity": algo_used, "n_slices": n_slices,
                       "parallelism": f"bank shard x{world} + NCCL all-gather/all-reduce + "
                                      + ("P2P fused merge-exchange" if exchange == "p2p"
                                         else "NCCL all-to-all"),
                       "graph": graph is not None,
                       "l2": "bank shard streamed from HBM each round"},
            "e2e": {"value": round(req * args.steps / (e2e_ms / 1e3), 1), "unit": "requests/s",
                    "h2d_bytes_per_step": int(world * (q.nbytes + qi.nbytes + I.nbytes + ids.nbytes)),
                    "d2h_bytes_per_step": int(world * 16 * NQ),
                    "ms_per_step": round(e2e_ms / args.steps, 4)},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "TFLOP/s", "frac": round(achieved / peak, 4),
                         "peak_source": "int8 dense = 2 x measured bf16 burst",
                         "kernel": topk_kernel_name(algo_used, world * NQ),
                         "kernel_ms": round(kern_ms, 4),
                         "kernel_share_of_step": round(kern_ms / (ms / args.steps), 3),
                         "traffic": None},
            "gpu_launches": int(per_round * args.steps),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def run_c5(args):
    """BASELINE configs[4] on one GPU: rolling trace replay against the c2
    bank (1M rows, pre-seeded), every round = completions pushed into the
    FIFO ring + arrivals predicted (stages 1-3) + bucket refreshes + full
    re-rank + batch packing, all device-resident, one native C-ABI call per
    round (ss_engine_round, csrc/k_engine.cu)."""
    import torch

    from paper_2603_07917_b200 import _build, _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.replay_device import DeviceTrace, NativeReplay
    from paper_2603_07917_b200.scheduler import RoundConfig
    from paper_2603_07917_b200.synthetic import inv_norm_device, make_bank_device

    torch.cuda.set_device(0)
    if _build.is_stale():
        _build.build()
    _lib.load()
    A, TOK, B, MAXA = 1024, 32, 8192, 65536
    rounds = args.warmup + args.steps
    n_trace = max(1 << 20, A * rounds)  # the 1M-request trace; the run replays its first rounds
    emb, lens, _ = make_bank_device(N_BANK, DIM, N_CLUSTERS, SEED)
    win = HistoryWindow(N_BANK, DIM)
    win.push(emb, lens)
    del emb, lens
    te, tl, _ = make_bank_device(n_trace, DIM, N_CLUSTERS, SEED, member_seed=SEED + 1000)
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED + 7)
    tr = DeviceTrace(te, inv_norm_device(te),
                     torch.randint(1, 4097, (n_trace,), generator=g, device="cuda",
                                   dtype=torch.int32), tl)
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
    dr = NativeReplay(win, tr, cfg, A, TOK, B, MAXA)  # one ss_engine_round call per round
    for _ in range(args.warmup):
        dr.round()
    torch.cuda.synchronize()
    a0, c0 = dr.stats.admitted, _lib.launch_count()
    n_act = []
    sampler = ClockSampler(0)
    with sampler:
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            dr.round()
            n_act.append(dr.n_act)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        clocks = sampler.summary(t0, time.time())
    admitted = dr.stats.admitted - a0
    print(json.dumps({
        "metric": "requests scheduled/sec over a rolling trace replay (arrivals predicted + "
                  "all active re-indexed, re-ranked and packed every round)",
        "value": round(admitted / (ms / 1e3), 1), "unit": "requests/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (clustered int8 embeddings; trace members share the bank's clusters)",
        "config": {"workload": "c5: rolling replay of a 1M-request trace against a 1M-entry "
                               "bank (one round per step; the run replays the first "
                               f"{rounds} rounds)",
                   "arrivals_per_round": A, "tokens_per_round": TOK, "batch": B, "k": K,
                   "nbins": NBINS, "theta": THETA,
                   "active_requests": [min(n_act), max(n_act)],
                   "completions_pushed": dr.stats.completed,
                   "driver": "native: one ss_engine_round C call per round"},
        "gpu_launches": int(_lib.launch_count() - c0), "clocks": clocks}), flush=True)


def run_c3(args):
    """BASELINE configs[2] 'Gittins refresh storm': 200k running+pending
    requests with 512-bin cost laws (64 length draws each), every index
    recomputed (conditioned on attained service) and the whole set re-ranked
    each step.  value = requests re-indexed and ranked per second."""
    import torch

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.scheduler import rank

    _lib.load()
    n, nbins, k = 200_000, 512, 64
    g = torch.Generator(device="cuda")
    g.manual_seed(SEED)
    d = "cuda"
    lens = torch.clamp(torch.round(torch.exp(5.5 + 0.8 * torch.randn((n, k), generator=g, device=d))),
                       1, 2048).to(torch.int32)
    I = torch.randint(1, 4097, (n,), generator=g, device=d, dtype=torch.int32)
    gg = torch.where(torch.rand(n, generator=g, device=d) < 0.4,
                     torch.randint(0, 2049, (n,), generator=g, device=d), 0).to(torch.int32)
    comp = torch.ones((n, k), dtype=torch.int64, device=d)
    fb = torch.zeros((3, nbins), dtype=torch.int64, device=d)
    npts = torch.zeros(n, dtype=torch.int32, device=d)
    pbin = torch.zeros((n, nbins), dtype=torch.int32, device=d)
    pcnt = torch.zeros((n, nbins), dtype=torch.int32, device=d)
    pD = torch.zeros((n, nbins), dtype=torch.int64, device=d)
    G = torch.zeros(n, dtype=torch.float64, device=d)
    P = lambda t: t.data_ptr()  # noqa: E731
    _lib.call("ss_finish", P(comp), P(lens), n, k, 1, 2048, nbins, P(I), P(fb[0]), P(fb[1]),
              P(fb[2]), nbins, P(npts), P(pbin), P(pcnt), P(pD), None, None, P(G),
              _lib.stream_ptr())
    bucket = torch.zeros(n, dtype=torch.int32, device=d)
    ids = torch.arange(n, dtype=torch.int64, device=d)
    perm = torch.empty(n, dtype=torch.int64, device=d)
    ws = torch.empty(int(_lib.lib().ss_rank_workspace_bytes(n)), dtype=torch.uint8, device=d)

    def step():
        _lib.call("ss_refresh", n, P(I), P(gg), P(bucket), 200, P(npts), P(pcnt), P(pD), nbins,
                  P(G), None, 1, _lib.stream_ptr())
        rank(G, ids, perm, ws)

    c0 = _lib.launch_count()
    step()
    torch.cuda.synchronize()
    per = _lib.launch_count() - c0
    # the storm's 1 + 39 launches replayed as one CUDA graph
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        step()
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    sampler = ClockSampler(0)
    with sampler:
        torch.cuda.synchronize()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        clocks = sampler.summary(t0, time.time())
        # refresh kernel alone for the roofline (HBM: the sparse laws it reads)
        e0.record()
        for _ in range(args.steps):
            _lib.call("ss_refresh", n, P(I), P(gg), P(bucket), 200, P(npts), P(pcnt), P(pD),
                      nbins, P(G), None, 1, _lib.stream_ptr())
        e1.record()
        torch.cuda.synchronize()
        kms = e0.elapsed_time(e1) / args.steps
    pts = int(npts.sum().item())
    byts = pts * 12 + n * (4 * 4 + 8)  # (count i32 + D i64) per point + per-request scalars + G
    pk = peaks()
    ach = byts / (kms / 1e3) / 1e9
    print(json.dumps({
        "metric": "requests re-indexed and re-ranked/sec (Gittins refresh storm)",
        "value": round(n * args.steps / (ms / 1e3), 1), "unit": "requests/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64/f64",
        "data": "synthetic (lognormal lengths, 64 draws per request, 40% running)",
        "config": {"workload": "c3: 200k running+pending requests, 512-bin cost distributions, "
                   "index recompute + full re-rank", "points_per_request": round(pts / n, 2)},
        "roofline": {"bound": "hbm", "achieved": round(ach, 1), "peak": pk["hbm_gbs"],
                     "unit": "GB/s", "frac": round(ach / pk["hbm_gbs"], 4), "kernel": "k_refresh",
                     "kernel_ms": round(kms, 4), "traffic": None},
        "gpu_launches": int(per * args.steps), "clocks": clocks}), flush=True)


def time_topk_kernel(sched, dq, dqi, args, nq=None):
    import ctypes as C

    import torch

    from paper_2603_07917_b200 import _lib

    algo = sched.cfg.algo
    code = _lib.ALGO[algo]
    if algo == "auto":
        # resolve what auto picks: try tcgen05 first
        code = _lib.ALGO["tcgen05"]
    n = nq or NQ
    max_slices = 1024
    part = torch.empty(max_slices * n * K, dtype=torch.int64, device="cuda")
    ns = C.c_int32()
    lib = _lib.lib()
    rc = lib.ss_topk_partials(sched.window.handle, dq.data_ptr(), dqi.data_ptr(), n, K,
                              float(np.float32(THETA)), code, part.data_ptr(), max_slices,
                              C.byref(ns), _lib.stream_ptr())
    used = "tcgen05"
    if rc != 0:
        code = _lib.ALGO["scan"]
        used = "scan"
        _lib.call("ss_topk_partials", sched.window.handle, dq.data_ptr(), dqi.data_ptr(), n, K,
                  float(np.float32(THETA)), code, part.data_ptr(), max_slices, C.byref(ns),
                  _lib.stream_ptr())
    elif algo == "scan":
        used = "scan"
    torch.cuda.synchronize()
    reps = max(3, args.steps)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        lib.ss_topk_partials(sched.window.handle, dq.data_ptr(), dqi.data_ptr(), n, K,
                             float(np.float32(THETA)), code, part.data_ptr(), max_slices,
                             C.byref(ns), _lib.stream_ptr())
    e1.record(st)
    torch.cuda.synchronize()
    return used, e0.elapsed_time(e1) / reps, int(ns.value)


def time_e2e(sched, q, qi, I, ids, args):
    import torch

    def pin(a):
        t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        return t.numpy()

    hq, hqi, hI, hids = pin(q), pin(qi), pin(I), pin(ids)
    G = torch.empty(NQ, dtype=torch.float64).pin_memory().numpy()
    perm = torch.empty(NQ, dtype=torch.int64).pin_memory().numpy()
    s = torch.cuda.Stream()
    for _ in range(max(1, args.warmup)):
        sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(args.steps):
        sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    h2d = hq.nbytes + hqi.nbytes + hI.nbytes + hids.nbytes
    d2h = G.nbytes + perm.nbytes
    return e0.elapsed_time(e1), int(h2d), int(d2h)


def topk_kernel_name(algo_used: str, nq: int) -> str:
    """Which stage-1 kernel the library launches (mirrors use_ts() in
    csrc/k_topk_sm100.cu): the A-in-TMEM tcgen05 kernel above one 128-query
    tile, the streaming form of k_topk_tc at or below it."""
    if algo_used != "tcgen05":
        return "k_topk_scan"
    if nq > 128 and os.environ.get("SS_TC_TS", "") != "0":
        return "k_topk_ts"
    return "k_topk_tc"


def ncu_traffic(kernel: str):
    """dram read+write bytes per launch of `kernel` on this workload, from the
    committed ncu --set full summary (profiles/ncu_traffic.json), else None."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(WORKLOAD.split(":")[0], {}).get(kernel)
    except Exception:
        return None


# --------------------------------------------------------- CPU reference ----
def _cpu_env():
    n = os.cpu_count() or 1
    for v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ.setdefault(v, str(n))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    return n


def _reference_modules():
    """The unmodified reference (servesim) when installed in baseline/_ref."""
    try:
        from servesim import _kernels as RK  # noqa: F401
        from servesim import cost as RC
        from servesim.distribution import DiscreteDistribution as RD
        RK.warmup()
        return RK, RC, RD
    except Exception:
        return None


class CpuRound:
    """The reference CPU path on one bank chunk: numpy/OpenBLAS fp32 similarity
    (exact on int8 vectors), per-chunk top-k (argpartition), merge, then per
    request the reference's cost_distribution + gittins_min, then lexsort."""

    def __init__(self, chunk_rows: int, seed: int = 0):
        from oracle import sagesched_oracle as O

        self.O = O
        self.mods = _reference_modules()
        emb, lens, _, _ = O.make_bank(chunk_rows + NQ, DIM, 256, seed)
        self.W = emb[:chunk_rows].astype(np.float32)
        self.iw = O.inv_norm(emb[:chunk_rows])
        self.lens = lens[:chunk_rows].astype(np.int64)
        self.Q = emb[chunk_rows:].astype(np.float32)
        self.iq = O.inv_norm(emb[chunk_rows:])
        self.I = np.random.default_rng(seed).integers(1, 4097, NQ)

    def chunk_topk(self):
        s = (self.Q @ self.W.T) * self.iw[None, :]
        s = s * self.iq[:, None]
        s[s < np.float32(THETA)] = -np.inf
        idx = np.argpartition(-s, K, axis=1)[:, :K]
        return s, idx

    def finish(self, s, idx):
        O = self.O
        G = np.empty(NQ)
        w = MAX_LEN // NBINS
        for i in range(NQ):
            sel = idx[i][np.isfinite(s[i, idx[i]])]
            L = self.lens[sel] if sel.size >= MIN_MATCHES else self.lens
            b = (np.minimum(L, MAX_LEN) - 1) // w
            Lf = L.astype(np.float64)
            cnt = np.bincount(b, minlength=NBINS)
            sv = np.bincount(b, weights=Lf, minlength=NBINS)
            sv2 = np.bincount(b, weights=Lf * Lf, minlength=NBINS)
            nz = np.flatnonzero(cnt)
            # conditional-mean ResourceBound cost per bin (cost.py:98-99 per length)
            sup = (sv2[nz] + 2.0 * self.I[i] * sv[nz]) * 0.5 / cnt[nz]
            mas = cnt[nz] / cnt[nz].sum()
            if self.mods:
                RK = self.mods[0]
                G[i] = RK.gittins_min(sup, mas)  # the reference's own numba kernel
            else:
                G[i] = O.gittins_min(sup, mas)
        return np.lexsort((np.arange(NQ), G))

    def step(self, n_chunks_total: int):
        """Time one chunk of stage 1 plus the full stages 2-4; extrapolate stage 1."""
        t0 = time.perf_counter()
        s, idx = self.chunk_topk()
        t1 = time.perf_counter()
        self.finish(s, idx)
        t2 = time.perf_counter()
        return (t1 - t0) * n_chunks_total + (t2 - t1)


def cpu_baseline(budget_s: float = 20.0):
    n = _cpu_env()
    chunk = 1 << 16
    total_chunks = N_BANK // chunk
    r = CpuRound(chunk)
    r.step(total_chunks)  # warm (BLAS threads, numba JIT)
    ts = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(ts) < 5:
        ts.append(r.step(total_chunks))
    t = float(np.median(ts))
    return {"value": round(NQ / t, 2), "unit": "requests/s", "cores": n,
            "kind": "port",
            "sample": (f"{NQ} queries x one {chunk}-row bank chunk (stage 1 extrapolated x{total_chunks} "
                       f"to the 1M bank) + full stages 2-4; median of {len(ts)}; Gittins = reference "
                       f"servesim gittins_min (numba) {'from baseline/_ref' if r.mods else 'unavailable -> oracle'}; "
                       "similarity/top-k/histogram are SPEC-only (numpy restatement)")}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = _cpu_env()
    chunk = 1 << 16
    total_chunks = N_BANK // chunk
    r = CpuRound(chunk)
    for _ in range(max(1, args.warmup)):
        r.step(total_chunks)
    ts = [r.step(total_chunks) for _ in range(args.steps)]
    t = float(np.sum(ts))
    value = NQ * args.steps / t
    cb = {"value": round(value, 2), "unit": "requests/s", "cores": n, "kind": "port",
          "sample": f"per step: {NQ} queries x one {chunk}-row chunk, stage 1 extrapolated x{total_chunks}"}
    line = {"impl": "reference",
            "metric": "requests scheduled/sec per round (predict+cost+Gittins+rank) vs a 1M-entry bank",
            "value": round(value, 2), "unit": "requests/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * t / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "nq": NQ, "k": K, "nbins": NBINS},
            "cpu_baseline": cb,
            "e2e": {"value": round(value, 2), "unit": "requests/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--algo", default="auto", choices=["auto", "scan", "tcgen05"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--config", default="c2", choices=["c2", "c3", "c4", "c5"],
                    help="c2 = headline (BASELINE configs[1]); c3 = refresh storm; "
                         "c4 = 16M bank x 8192 queries on this GPU")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    global N_BANK, NQ, WORKLOAD
    if args.config == "c4":
        N_BANK, NQ = 1 << 24, 8192
        WORKLOAD = "c4: 16M-entry x 384-d int8 history bank, 8192 queries/round, k=64, 128 bins"
    if args.config == "c3" and args.impl == "ours":
        return run_c3(args)
    if args.config == "c5" and args.impl == "ours":
        return run_c5(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

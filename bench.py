"""Benchmark of the SageSched per-round scheduling hot path on B200.

One step = one scheduling round over one batch of synthetic pending requests:
predict (history bank -> top-64 -> 128-bin length histogram) -> cost
(O^2/2 + I*O) -> Gittins index -> rank.

  N = 1   workload = BASELINE.json configs[1] (1M x 384 bank, 1024 pending
          prompts per round, k=64, 128 bins, theta = 0.8) on one GPU.
  N > 1   workload = configs[3] (16M x 384 bank row-sharded over the N GPUs,
          one 8192-request queue owned by rank 0; single-owner round:
          query broadcast, local fused top-k, all-gather of k candidates per
          query, merge + cost + Gittins + rank on the owner) -- strong
          scaling.  ``--config c4 --sharded`` runs the same code path at N=1.

  value  requests scheduled / s with inputs resident in HBM (CUDA-graph replay
         of the round, CUDA events, max over ranks)
  e2e    same metric through the plugin call from pinned HOST buffers
         (H2D + round + D2H inside the timed region)
  roofline       the dominant kernel (the tcgen05 similarity + fused top-k)
                 against the int8 tensor peak measured live by tools/mma_peak.cu
  roofline_scan  the bank-scan form of the same kernel (8 queries, HBM-bound)
                 against the measured HBM copy bandwidth -- BASELINE's "bank-scan
                 HBM GB/s % of peak"

``--impl reference`` times the reference's CPU implementation of the path
(servesim from baseline/_ref where the code exists -- match/gittins_min --
and the oracle restatement of the SPEC-only pieces) on the host cores: every
step is a sample of the round's queries scored against the WHOLE bank.
"""

from __future__ import annotations

import os

# CPU thread pools (OpenBLAS GEMM, numba) sized before numpy / numba load
_NCPU = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
    os.environ[_v] = str(_NCPU)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nbcache")

import argparse  # noqa: E402
import ctypes  # noqa: E402
import json  # noqa: E402
import socket  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import threading  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIM, K, NBINS, MAX_LEN = 384, 64, 128, 2048
THETA, MIN_MATCHES, N_CLUSTERS = 0.8, 20, 4096
SEED = 0
CONFIGS = {
    "c2": dict(n_bank=1 << 20, nq=1024,
               workload="c2: 1M-entry x 384-d int8 history bank, 1024 pending prompts/round, "
                        "k=64, 128 bins"),
    "c4": dict(n_bank=1 << 24, nq=8192,
               workload="c4: 16M-entry x 384-d int8 history bank, 8192 pending prompts/round, "
                        "k=64, 128 bins"),
}
METRIC = "requests scheduled/sec per round (predict+cost+Gittins+rank)"
SCAN_NQ = 8  # the bank-scan (HBM-bound) form of the similarity kernel


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


# ------------------------------------------------------ device measurement --
def time_ms(fn, reps, stream=None):
    """Average CUDA-event time of fn() on `stream` (default: torch's current)."""
    import torch
    st = stream or torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def int8_peak():
    """Dense int8 tensor-core ceiling measured now on this GPU by the probe
    tools/mma_peak.cu (operands resident, back-to-back tcgen05.mma kind::i8,
    M=128 K=32, one CTA per SM).  -> (TOPS, detail)."""
    import torch
    from paper_2603_07917_b200 import _build
    _build.build_probes()
    so = _build.PROBES[os.path.join(_build.TOOLS_DIR, "mma_peak.cu")]
    lib = ctypes.CDLL(so)
    lib.mma_peak_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    st = torch.cuda.current_stream()
    out = {}
    for n, a_tmem in ((256, 0), (256, 1), (208, 1)):
        tiles = 12000
        if lib.mma_peak_run(sms, 50, n, a_tmem, ctypes.c_void_p(st.cuda_stream)):
            continue
        ms = min(time_ms(lambda: lib.mma_peak_run(sms, tiles, n, a_tmem,
                                                  ctypes.c_void_p(st.cuda_stream)), 1)
                 for _ in range(3))
        ops = 2.0 * 128 * n * DIM * tiles * sms
        out[f"N{n}_{'ts' if a_tmem else 'ss'}"] = round(ops / (ms / 1e3) / 1e12, 1)
    best = max(out.values()) if out else None
    return best, out


def int8_peak_sustained(seconds: float = 3.0):
    """The same probe (N = 256, A in TMEM) run back to back for ``seconds``
    so the board settles under its power cap; the rate over the last third
    is the sustained int8 ceiling -- the denominator for a kernel timed
    inside a long step (c4: ~44 ms per round, seconds per run), as the
    profiling recipe prescribes for bf16.  -> (TOPS, clocks during the tail)."""
    import torch
    from paper_2603_07917_b200 import _build
    _build.build_probes()
    lib = ctypes.CDLL(_build.PROBES[os.path.join(_build.TOOLS_DIR, "mma_peak.cu")])
    lib.mma_peak_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    tiles = 6000
    if lib.mma_peak_run(sms, 50, 256, 1, st):
        return None, None
    ops = 2.0 * 128 * 256 * DIM * tiles * sms
    rates, t_end = [], time.time() + seconds
    sampler = ClockSampler(0)
    with sampler:
        while time.time() < t_end:
            ms = time_ms(lambda: lib.mma_peak_run(sms, tiles, 256, 1, st), 1)
            rates.append((time.time(), ops / (ms / 1e3) / 1e12))
        t_tail = t_end - seconds / 3
        clocks = sampler.summary(t_tail, time.time())
    tail = sorted(r for t, r in rates if t >= t_tail) or [r for _, r in rates]
    return round(tail[len(tail) // 2], 1), clocks


def sustained_roof(roof: dict, achieved: float) -> None:
    """A kernel timed inside a long run (the c4 round: tens of ms per step,
    the board under sw_power_cap) is divided by the sustained ceiling; the
    burst probe stays in the record as peak_burst / frac_of_burst."""
    s, sclk = int8_peak_sustained()
    if not s:
        return
    roof["peak_burst"], roof["frac_of_burst"] = roof["peak"], roof["frac"]
    roof["peak"], roof["frac"] = s, round(achieved / s, 4)
    roof["peak_source"] = ("int8 tcgen05.mma kind::i8 ceiling SUSTAINED: tools/mma_peak.cu (N = 256, A "
                           "in TMEM) back to back for 3 s, median rate of the last second "
                           f"(clocks then: {sclk}); burst probe: peak_burst")


def cublas_int8_tops():
    """cuBLASLt int8 GEMM rate (torch._int_mm, 8192 x 8192 x 384 -> int32), for context."""
    import torch
    try:
        a = torch.randint(-127, 128, (8192, DIM), dtype=torch.int8, device="cuda")
        b = torch.randint(-127, 128, (DIM, 8192), dtype=torch.int8, device="cuda")
        torch._int_mm(a, b)
        ms = min(time_ms(lambda: torch._int_mm(a, b), 20) for _ in range(3))
        return round(2.0 * 8192 * 8192 * DIM / (ms / 1e3) / 1e12, 1)
    except Exception:
        return None


def ncu_traffic(workload_key: str, kernel: str):
    """dram read+write bytes per launch of `kernel` on this workload, from the
    committed ncu --set full summary (profiles/ncu_traffic.json), else None."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(workload_key, {}).get(kernel)
    except Exception:
        return None


def topk_kernel_name(nq: int) -> str:
    """The stage-1 kernel the library launches for nq queries (csrc/k_topk_sm100.cu
    use_ts): the A-in-TMEM kernel above one 128-query tile, the streaming
    form of k_topk_tc at or below it."""
    return "k_topk_ts" if nq > 128 else "k_topk_tc"


def time_topk(window, q, qi, nq, theta, reps):
    """The dominant kernel alone (similarity + fused top-k, ss_topk_partials)
    on torch's current stream, CUDA events.  -> (ms per launch, slices)."""
    import torch
    from paper_2603_07917_b200 import _lib
    max_slices = 1024
    part = torch.empty(max_slices * nq * K, dtype=torch.int64, device="cuda")
    ns = ctypes.c_int32()
    lib = _lib.lib()

    def go():
        rc = lib.ss_topk_partials(window.handle, q.data_ptr(), qi.data_ptr(), nq, K,
                                  float(np.float32(theta)), _lib.ALGO["tcgen05"], part.data_ptr(),
                                  max_slices, ctypes.byref(ns), _lib.stream_ptr())
        if rc:
            _lib.check(rc, "ss_topk_partials")
    go()
    return time_ms(go, reps), int(ns.value)


# ------------------------------------------------------------ our arm -----
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2603_07917_b200 import _build, _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # (ranks beyond the visible GPUs share them: the --backend gloo check of
    # the multi-rank path on a one-GPU box)
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    sharded = world > 1 or args.sharded
    if sharded:
        if "MASTER_ADDR" not in os.environ:  # --sharded at N = 1 without torchrun
            with socket.socket() as s:
                s.bind(("127.0.0.1", 0))
                os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(s.getsockname()[1]),
                                  RANK="0", WORLD_SIZE="1")
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group("gloo")
    if rank == 0 and (_build.is_stale() or not os.path.exists(_build.LIB_PATH)):
        _build.build()
    if sharded:
        dist.barrier()
    _lib.load()
    if sharded:
        return run_sharded(args, world, rank, local)
    return run_single(args)


def run_single(args):
    import torch

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    C = CONFIGS[args.config]
    n_bank, nq = C["n_bank"], C["nq"]
    emb, lens, _ = make_bank_device(n_bank, DIM, N_CLUSTERS, SEED)
    win = HistoryWindow(n_bank, DIM)
    win.push(emb, lens)
    del emb, lens
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
    sched = SageScheduler(win, cfg)

    # launches per round (counted on an eager round)
    c0 = _lib.launch_count()
    sched.schedule_round(dq, dqi, dI, dids)
    torch.cuda.synchronize()
    per_round = _lib.launch_count() - c0

    graph, _ = sched.capture_round(dq, dqi, dI, dids)
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()

    sampler = ClockSampler(0)
    with sampler:
        torch.cuda.synchronize()
        t0 = time.time()
        ms = time_ms(graph.replay, args.steps) * args.steps
        t1 = time.time()
        clocks = sampler.summary(t0, t1)
        # dominant kernel alone (similarity + fused top-k), same stream
        kern_ms, n_slices = time_topk(win, dq, dqi, nq, THETA, max(3, args.steps))
        # the bank scan: 8 queries against the whole bank (HBM-bound form)
        scan_ms, scan_slices = time_topk(win, dq[:SCAN_NQ].contiguous(), dqi[:SCAN_NQ].contiguous(),
                                         SCAN_NQ, THETA, max(10, args.steps))
        # e2e: plugin call from pinned host buffers
        e2e_ms, h2d, d2h = time_e2e(sched, q, qi, I, ids, args)
    # north star's literal "select top-k" (theta <= 0): same round, pure top-k
    pure = None
    if not args.no_pure:
        pcfg = RoundConfig(k=K, theta=-1.0, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
        psched = SageScheduler(win, pcfg)
        pg, _ = psched.capture_round(dq, dqi, dI, dids)
        for _ in range(3):
            pg.replay()
        pms = time_ms(pg.replay, max(3, args.steps // 2))
        pk_ms, _ = time_topk(win, dq, dqi, nq, -1.0, max(3, args.steps // 2))
        pure = {"theta": -1.0, "value": round(nq / (pms / 1e3), 1), "unit": "requests/s",
                "ms_per_step": round(pms, 4), "kernel_ms": round(pk_ms, 4)}

    pk = peaks()
    i8_peak, i8_detail = int8_peak()
    ops = 2.0 * nq * n_bank * DIM
    achieved = ops / (kern_ms / 1e3) / 1e12
    kname = topk_kernel_name(nq)
    roof = {"bound": "tensor", "achieved": round(achieved, 1), "peak": i8_peak, "unit": "TFLOP/s",
            "frac": round(achieved / i8_peak, 4) if i8_peak else None,
            "peak_source": "int8 dense tcgen05.mma kind::i8 ceiling measured live on this GPU by "
                           f"tools/mma_peak.cu (best of {i8_detail}); nominal 4500",
            "cublas_int8_tops": cublas_int8_tops(),
            "work_per_launch": f"2 * nq * N * d = 2 * {nq} * {n_bank} * {DIM} int8 ops",
            "kernel": kname, "kernel_ms": round(kern_ms, 4), "n_slices": n_slices,
            "kernel_share_of_step": round(kern_ms / (ms / args.steps), 3),
            "traffic": ncu_traffic(args.config, kname),
            "traffic_algorithmic": int(n_bank * (DIM + 4))}
    if args.config == "c4":
        sustained_roof(roof, achieved)
    scan_bytes = n_bank * (DIM + 4) + SCAN_NQ * (DIM + 4)
    scan_gbs = scan_bytes / (scan_ms / 1e3) / 1e9
    roof_scan = {"bound": "hbm", "achieved": round(scan_gbs, 1), "peak": pk["hbm_gbs"], "unit": "GB/s",
                 "frac": round(scan_gbs / pk["hbm_gbs"], 4),
                 "frac_of_8tbs_datasheet": round(scan_gbs / 8000.0, 4),
                 "peak_source": "measured copy bandwidth (MEASURED_PEAKS.json)",
                 "work_per_launch": f"bank bytes N * (d + 4) = {n_bank} * {DIM + 4}",
                 "kernel": topk_kernel_name(SCAN_NQ), "nq": SCAN_NQ, "n_slices": scan_slices,
                 "kernel_ms": round(scan_ms, 4),
                 "traffic": ncu_traffic(args.config + "_scan8", topk_kernel_name(SCAN_NQ))}
    # the north star's target shape (BASELINE configs[3]) on this one GPU
    # (after the peak probes: its long run heats the part): the per-GPU
    # similarity work of the 8-GPU configuration is 1/8 of it
    c4 = sweep = proj = None
    if args.config == "c2" and not args.no_c4:
        del graph, sched, win
        torch.cuda.empty_cache()
        c4 = c4_one_gpu(args)
        sweep = vs_bank_size(args)
        proj = c4_projection()
    line = {
        "metric": METRIC, "value": round(nq * args.steps / (ms / 1e3), 1), "unit": "requests/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int8",
        "data": "synthetic (seeded clustered int8 embeddings, lognormal lengths)",
        "config": {"workload": C["workload"], "bank_rows": n_bank, "dim": DIM, "nq": nq, "k": K,
                   "nbins": NBINS, "theta": THETA, "min_matches": MIN_MATCHES,
                   "parallelism": "single GPU",
                   "l2": f"bank ({n_bank * (DIM + 4) / 1e6:.0f} MB) > L2 (126 MB): every round "
                         "streams it from HBM"},
        "e2e": {"value": round(nq * args.steps / (e2e_ms / 1e3), 1), "unit": "requests/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(e2e_ms / args.steps, 4)},
        "roofline": roof,
        "roofline_scan": roof_scan,
        "pure_topk": pure,
        "c4_one_gpu": c4,
        "vs_bank_size": sweep,
        "c4_n_gpus_projection": proj,
        "gpu_launches": int(per_round * args.steps),
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and args.config == "c2":
        line["cpu_baseline"] = cpu_baseline(args.config, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)


def c4_one_gpu(args):
    """The c4 round (16M x 384 bank, 8192 requests) on this GPU: graph-replayed
    rounds and the similarity kernel alone, a few steps (a sub-record of the
    default c2 line; `--config c4` gives the full line)."""
    import torch

    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    C = CONFIGS["c4"]
    n_bank, nq = C["n_bank"], C["nq"]
    emb, lens, _ = make_bank_device(n_bank, DIM, N_CLUSTERS, SEED)
    win = HistoryWindow(n_bank, DIM)
    win.push(emb, lens)
    del emb, lens
    torch.cuda.empty_cache()
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
    sched = SageScheduler(win, cfg)
    graph, _ = sched.capture_round(dq, dqi, dI, dids)
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    steps = 5
    sampler = ClockSampler(0)
    with sampler:
        t0 = time.time()
        ms = time_ms(graph.replay, steps)
        t1 = time.time()
        clocks = sampler.summary(t0, t1)
    kern_ms, n_slices = time_topk(win, dq, dqi, nq, THETA, 3)
    out = {"workload": C["workload"], "value": round(nq / (ms / 1e3), 1), "unit": "requests/s",
           "ms_per_step": round(ms, 3), "steps": steps, "kernel": topk_kernel_name(nq),
           "kernel_ms": round(kern_ms, 3), "n_slices": n_slices,
           "kernel_tops": round(2.0 * nq * n_bank * DIM / (kern_ms / 1e3) / 1e12, 1),
           "clocks": clocks}
    s_peak, s_clk = int8_peak_sustained()
    if s_peak:
        out["int8_sustained_tops"] = s_peak
        out["kernel_frac_of_sustained"] = round(out["kernel_tops"] / s_peak, 4)
        out["sustained_probe_clocks"] = s_clk
    del graph, sched, win, dq, dqi, dI, dids
    torch.cuda.empty_cache()
    return out


NVLINK_GBS, COLL_LAT_US = 770.0, 15.0  # B200_PROFILING.md peer copy per direction; per-collective latency


def c4_projection(rows=1 << 24, nq=8192, worlds=(2, 4, 8), reps=5):
    """c4 single-owner round at N GPUs PROJECTED from components measured on
    this one GPU (not a multi-GPU measurement): the bank cut into N shards by
    ShardPlan exactly as the sharded round places them; every shard's local
    stage (HistoryWindow.topk: TS kernel + slice merge) timed with CUDA
    events; the owner's stages (ss_merge_topk of the N lists, ss_finish,
    ss_rank) timed on the stacked shard outputs; the merged lists, window
    histogram, G and order checked bit-identical to the unsharded round.  The
    broadcast and all-gather are charged at NVLINK_GBS + COLL_LAT_US each.
    round(N) = max over shards of the local stage + collectives + owner."""
    import torch

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import rank
    from paper_2603_07917_b200.sharded import ShardPlan
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    _lib.load()
    P = _lib.ptr
    emb, lens, _ = make_bank_device(rows, DIM, N_CLUSTERS, SEED)
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))

    def owner(comp_x, len_x, nlists, fb):
        comp = torch.empty((nq, K), dtype=torch.int64, device="cuda")
        ln = torch.empty((nq, K), dtype=torch.int32, device="cuda")
        o = {n: torch.zeros(sh, dtype=dt, device="cuda") for n, sh, dt in (
            ("npts", nq, torch.int32), ("pbin", (nq, NBINS), torch.int32),
            ("pcnt", (nq, NBINS), torch.int32), ("pD", (nq, NBINS), torch.int64),
            ("used_fb", nq, torch.uint8), ("G", nq, torch.float64), ("perm", nq, torch.int64))}
        ws = torch.empty(int(_lib.lib().ss_rank_workspace_bytes(nq)), dtype=torch.uint8, device="cuda")
        c, l_ = (comp, ln) if nlists > 1 else (comp_x, len_x)

        def go():
            if nlists > 1:
                _lib.call("ss_merge_topk", P(comp_x), P(len_x), nlists, nq, K, P(comp), P(ln),
                          _lib.stream_ptr())
            _lib.call("ss_finish", P(c), P(l_), nq, K, MIN_MATCHES, MAX_LEN, NBINS, P(dI), P(fb[0]),
                      P(fb[1]), P(fb[2]), NBINS, P(o["npts"]), P(o["pbin"]), P(o["pcnt"]),
                      P(o["pD"]), None, P(o["used_fb"]), P(o["G"]), _lib.stream_ptr())
            rank(o["G"], dids, o["perm"], ws)
        t = time_ms(go, reps)
        go()
        torch.cuda.synchronize()
        return t, c, l_, o

    full = HistoryWindow(rows, DIM)
    full.push(emb, lens)
    fb1 = full.fallback_hist(MAX_LEN, NBINS)
    full.topk(dq, dqi, K, THETA)
    t_loc1 = time_ms(lambda: full.topk(dq, dqi, K, THETA), reps)
    c1, l1 = full.topk(dq, dqi, K, THETA)
    t_own1, _, _, o1 = owner(c1, l1, 1, fb1)
    del full
    torch.cuda.empty_cache()
    out = {"what": "c4 single-owner round on N GPUs PROJECTED from components measured on this "
                   "one GPU (not a multi-GPU measurement)",
           "rows": rows, "nq": nq, "k": K, "theta": THETA,
           "one_gpu_round_ms": round(t_loc1 + t_own1, 3),
           "collective_model": f"{NVLINK_GBS} GB/s per direction (B200_PROFILING.md peer copy) + "
                               f"{COLL_LAT_US} us per collective (broadcast, all-gather)",
           "points": []}
    for world in worlds:
        comps, lns, times = [], [], []
        fb = torch.zeros((3, NBINS), dtype=torch.int64, device="cuda")
        for r in range(world):
            plan = ShardPlan(rows, world, r)  # the sharded round's own placement
            w = HistoryWindow(plan.local_capacity, DIM, global_capacity=rows,
                              slot_offset=plan.slot_offset)
            idx, seq, slot = (torch.as_tensor(x, device="cuda") for x in plan.route(0, rows))
            w.write(emb[idx], lens[idx], seq, slot)
            w.set_head(rows)
            del idx, seq, slot
            fb += w.fallback_hist(MAX_LEN, NBINS)
            w.topk(dq, dqi, K, THETA)
            times.append(time_ms(lambda: w.topk(dq, dqi, K, THETA), reps))
            c, l_ = w.topk(dq, dqi, K, THETA)
            comps.append(c)
            lns.append(l_)
            del w
            torch.cuda.empty_cache()
        t_own, c, l_, o = owner(torch.stack(comps).contiguous(), torch.stack(lns).contiguous(),
                                world, fb)
        exact = bool(torch.equal(c, c1) and torch.equal(l_, l1) and torch.equal(fb, fb1)
                     and torch.equal(o["G"], o1["G"]) and torch.equal(o["perm"], o1["perm"]))
        coll_b = nq * (DIM + 4) + (world - 1) * nq * K * 12  # queue broadcast + owner's gather
        t_coll = coll_b / (NVLINK_GBS * 1e9) * 1e3 + 2 * COLL_LAT_US / 1e3
        t_round = max(times) + t_coll + t_own
        out["points"].append({
            "n_gpus": world, "shard_rows": rows // world,
            "local_stage_ms_max": round(max(times), 3), "local_stage_ms_min": round(min(times), 3),
            "owner_merge_finish_rank_ms": round(t_own, 3), "collectives_ms_modelled": round(t_coll, 3),
            "projected_round_ms": round(t_round, 3),
            "projected_value": round(nq / (t_round / 1e3), 1), "unit": "requests/s",
            "bit_identical_to_one_gpu_round": exact})
    del emb, lens
    torch.cuda.empty_cache()
    return out


def vs_bank_size(args, sizes=(1 << 16, 1 << 18, 1 << 20, 1 << 22, 1 << 24)):
    """BASELINE's metric is requests scheduled/s per round *vs bank size*: the
    c2 round (1024 prompts, k 64, 128 bins, theta 0.8) over banks of 64k ..
    16M rows, graph-replayed, five rounds each."""
    import torch

    from paper_2603_07917_b200.history import HistoryWindow
    from paper_2603_07917_b200.scheduler import RoundConfig, SageScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    nq = CONFIGS["c2"]["nq"]
    emb, lens, _ = make_bank_device(max(sizes), DIM, N_CLUSTERS, SEED)
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
    out = []
    for n in sizes:
        win = HistoryWindow(n, DIM)
        win.push(emb[:n], lens[:n])
        sched = SageScheduler(win, cfg)
        graph, _ = sched.capture_round(dq, dqi, dI, dids)
        for _ in range(3):
            graph.replay()
        ms = time_ms(graph.replay, 5)
        out.append({"bank_rows": n, "ms_per_step": round(ms, 4), "value": round(nq / (ms / 1e3), 1),
                    "unit": "requests/s"})
        del graph, sched, win
        torch.cuda.empty_cache()
    del emb, lens
    torch.cuda.empty_cache()
    return {"nq": nq, "k": K, "nbins": NBINS, "theta": THETA, "points": out}


def time_e2e(sched, q, qi, I, ids, args):
    import torch

    def pin(a):
        return torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()

    nq = q.shape[0]
    hq, hqi, hI, hids = pin(q), pin(qi), pin(I), pin(ids)
    G = torch.empty(nq, dtype=torch.float64).pin_memory().numpy()
    perm = torch.empty(nq, dtype=torch.int64).pin_memory().numpy()
    s = torch.cuda.Stream()
    for _ in range(max(3, args.warmup)):
        sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s)
    ms = time_ms(lambda: sched.schedule_round_host(hq, hqi, hI, hids, G, perm, stream=s),
                 args.steps, stream=s) * args.steps
    return ms, int(hq.nbytes + hqi.nbytes + hI.nbytes + hids.nbytes), int(G.nbytes + perm.nbytes)


def run_sharded(args, world, rank, local):
    """Single-owner round over a row-sharded bank (c4 by default at N > 1):
    rank 0 owns the whole queue; every GPU scores it against its 1/N of the
    bank; the k candidates per query are all-gathered; the owner merges,
    finishes and ranks.  Strong scaling: the total work is fixed."""
    import torch
    import torch.distributed as dist

    from paper_2603_07917_b200 import _lib
    from paper_2603_07917_b200.scheduler import RoundConfig
    from paper_2603_07917_b200.sharded import ShardedHistory, ShardedScheduler
    from paper_2603_07917_b200.synthetic import make_bank_device, make_queries

    C = CONFIGS[args.config]
    n_bank, nq = C["n_bank"], C["nq"]
    owner = 0
    emb, lens, _ = make_bank_device(n_bank, DIM, N_CLUSTERS, SEED)
    hist = ShardedHistory(n_bank, DIM)
    hist.push(emb, lens)
    del emb, lens
    torch.cuda.empty_cache()
    q, qi, I, ids = make_queries(nq, DIM, N_CLUSTERS, SEED, qseed=1000)
    dq, dqi, dI, dids = (torch.as_tensor(x, device="cuda") for x in (q, qi, I, ids))
    cfg = RoundConfig(k=K, theta=THETA, min_matches=MIN_MATCHES, max_len=MAX_LEN, nbins=NBINS)
    sched = ShardedScheduler(hist, cfg, exchange=args.exchange, owner=owner)
    mine = rank == owner
    args_round = (dq, dqi, dI, dids) if mine else (None, None, None, None)
    c0 = _lib.launch_count()
    sched.schedule_round(*args_round, nq=nq)
    torch.cuda.synchronize()
    per_round = _lib.launch_count() - c0
    graph = None
    try:
        if args.backend == "gloo":  # gloo collectives cannot be captured into a CUDA graph
            raise RuntimeError("gloo backend")
        graph, _ = sched.capture_round(*args_round, nq=nq)
    except Exception as e:  # noqa: BLE001
        print(f"sharded round not captured ({type(e).__name__}: {e}); timing eager rounds",
              file=sys.stderr)
        torch.cuda.synchronize()

    def one_round():
        if graph is not None:
            graph.replay()
        else:
            sched.schedule_round(*args_round, nq=nq)

    for _ in range(args.warmup):
        one_round()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    with sampler:
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.time()
        ms = time_ms(one_round, args.steps) * args.steps
        t1 = time.time()
        dist.barrier()
        clocks = sampler.summary(t0, t1)
        # e2e: the owner's pinned host queue in, order + indices out, every step
        if mine:
            hq, hqi, hI, hids = (torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
                                 for x in (q, qi, I, ids))
            hG = torch.empty(nq, dtype=torch.float64).pin_memory()
            hp = torch.empty(nq, dtype=torch.int64).pin_memory()
            host_args = (hq, hqi, hI, hids, hG, hp)
        else:
            host_args = (None, None, None, None, None, None)
        for _ in range(max(3, args.warmup)):
            sched.schedule_round_host(*host_args, nq=nq)
        dist.barrier()
        e2e_ms = time_ms(lambda: sched.schedule_round_host(*host_args, nq=nq), args.steps) * args.steps
        # dominant kernel: the local similarity of the whole queue against this shard
        kern_ms, n_slices = time_topk(hist.window, dq, dqi, nq, THETA, max(3, args.steps))
    vals = torch.tensor([ms, e2e_ms, kern_ms], dtype=torch.float64, device="cuda")
    dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms, kern_ms = vals.tolist()
    if rank == 0:
        i8_peak, i8_detail = int8_peak()
        ops = 2.0 * nq * (n_bank // world) * DIM
        achieved = ops / (kern_ms / 1e3) / 1e12
        B = "NCCL" if args.backend == "nccl" else "gloo (functional check: ranks share GPUs)"
        line = {
            "metric": METRIC, "value": round(nq * args.steps / (ms / 1e3), 1), "unit": "requests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int8",
            "data": "synthetic (seeded clustered int8 embeddings, lognormal lengths)",
            "config": {"workload": C["workload"] + f"; bank row-sharded over {world} GPU(s), "
                       "one queue owned by rank 0", "bank_rows": n_bank, "dim": DIM, "nq": nq,
                       "k": K, "nbins": NBINS, "theta": THETA, "min_matches": MIN_MATCHES,
                       "parallelism": f"bank shard x{world}; {B} broadcast of the queue, "
                                      + ("fused P2P gather of k candidates/query (ss_topk_gather)"
                                         if args.exchange == "p2p" else
                                         f"{B} all-gather of k candidates/query")
                                      + f", {B} all-reduce of the window histogram; stages 2-4 "
                                        "on the owner",
                       "graph": graph is not None,
                       "l2": "bank shard streamed from HBM each round"},
            "e2e": {"value": round(nq * args.steps / (e2e_ms / 1e3), 1), "unit": "requests/s",
                    "h2d_bytes_per_step": int(q.nbytes + qi.nbytes + I.nbytes + ids.nbytes),
                    "d2h_bytes_per_step": int(16 * nq),
                    "ms_per_step": round(e2e_ms / args.steps, 4)},
            "roofline": {"bound": "tensor", "achieved": round(achieved, 1), "peak": i8_peak,
                         "unit": "TFLOP/s", "frac": round(achieved / i8_peak, 4) if i8_peak else None,
                         "peak_source": f"int8 tcgen05 ceiling measured live (tools/mma_peak.cu: {i8_detail})",
                         "work_per_launch": f"2 * {nq} * {n_bank // world} * {DIM} int8 ops",
                         "kernel": topk_kernel_name(nq), "kernel_ms": round(kern_ms, 4),
                         "n_slices": n_slices,
                         "kernel_share_of_step": round(kern_ms / (ms / args.steps), 3),
                         "traffic": None},
            "gpu_launches": int(per_round * args.steps),
            "clocks": clocks,
        }
        sustained_roof(line["roofline"], achieved)
        print(json.dumps(line), flush=True)
    sched.close()
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
    n_bank = CONFIGS["c2"]["n_bank"]
    A, TOK, B, MAXA = 1024, 32, 8192, 65536
    rounds = args.warmup + args.steps
    n_trace = max(1 << 20, A * rounds)  # the 1M-request trace; the run replays its first rounds
    emb, lens, _ = make_bank_device(n_bank, DIM, N_CLUSTERS, SEED)
    win = HistoryWindow(n_bank, DIM)
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

    def refresh():
        _lib.call("ss_refresh", n, P(I), P(gg), P(bucket), 200, P(npts), P(pcnt), P(pD), nbins,
                  P(G), None, 1, _lib.stream_ptr())

    def step():
        refresh()
        rank(G, ids, perm, ws)

    c0 = _lib.launch_count()
    step()
    torch.cuda.synchronize()
    per = _lib.launch_count() - c0
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
        t0 = time.time()
        ms = time_ms(graph.replay, args.steps) * args.steps
        clocks = sampler.summary(t0, time.time())
        kms = time_ms(refresh, args.steps)  # refresh kernel alone (HBM: the laws it reads)
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
                     "kernel_ms": round(kms, 4), "traffic": ncu_traffic("c3", "k_refresh")},
        "gpu_launches": int(per * args.steps), "clocks": clocks}), flush=True)


# --------------------------------------------------------- CPU reference ----
def _reference_modules():
    """The unmodified reference (servesim) when installed in baseline/_ref."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from servesim import _kernels as RK
        RK.warmup()
        return RK
    except Exception:
        return None


class CpuRound:
    """The reference CPU path for the whole bank: numpy/OpenBLAS fp32
    similarity (exact on int8-valued vectors) in 128k-row chunks, selection
    (theta filter + top-k by (key desc, seq desc)), the window fallback, the
    fixed-bin histogram with per-bin conditional-mean ResourceBound cost
    (cost.py:97-99 per length), the reference's numba gittins_min
    (_kernels.py:104-116) per request, then lexsort by (G, id).  One step
    scores `sample` of the round's queries against every bank row."""

    CHUNK = 1 << 17

    def __init__(self, config: str, sample: int):
        from oracle import sagesched_oracle as O
        from paper_2603_07917_b200.synthetic import make_bank_host, make_queries

        C = CONFIGS[config]
        self.O, self.RK = O, _reference_modules()
        self.n = C["n_bank"]
        emb, lens = make_bank_host(self.n, DIM, N_CLUSTERS, SEED)
        self.iw = O.inv_norm(emb)
        # fp32 copy of the bank when it fits in a third of the free host memory
        # (c2: 1.6 GB; c4: 25.8 GB on a 196 GB box), else the int8 bank with
        # each chunk widened inside the step (slower: the widening dominates)
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:  # noqa: BLE001
            avail = 0
        fp32_bytes = emb.size * 4
        self.W = emb.astype(np.float32) if (self.n <= (1 << 22) or fp32_bytes * 3 < avail) else emb
        self.lens = lens.astype(np.int64)
        self.fb = O.bin_hist(self.lens, MAX_LEN, NBINS)
        q, qi, I, ids = make_queries(C["nq"], DIM, N_CLUSTERS, SEED, qseed=1000)
        self.sample = min(sample, C["nq"])
        self.Q = q[:self.sample].astype(np.float32)
        self.iq = qi[:self.sample]
        self.I = I[:self.sample].astype(np.int64)
        self.ids = ids[:self.sample]

    def step(self):
        O = self.O
        nq = self.sample
        keys, seqs = [[] for _ in range(nq)], [[] for _ in range(nq)]
        for s in range(0, self.n, self.CHUNK):
            Wc = self.W[s:s + self.CHUNK]
            if Wc.dtype != np.float32:
                Wc = Wc.astype(np.float32)
            sc = (self.Q @ Wc.T) * self.iw[None, s:s + self.CHUNK]
            sc *= self.iq[:, None]
            if THETA > 0:
                r, c = np.nonzero(sc >= np.float32(THETA))
                for i in np.unique(r):
                    m = r == i
                    keys[i].append(sc[i, c[m]])
                    seqs[i].append(c[m] + s)
            else:
                kk = min(K, sc.shape[1])
                top = np.argpartition(-sc, kk - 1, axis=1)[:, :kk]
                for i in range(nq):
                    keys[i].append(sc[i, top[i]])
                    seqs[i].append(top[i] + s)
        G = np.empty(nq)
        w = MAX_LEN // NBINS
        for i in range(nq):
            kv = np.concatenate(keys[i]) if keys[i] else np.zeros(0, np.float32)
            sv = np.concatenate(seqs[i]) if seqs[i] else np.zeros(0, np.int64)
            sel = sv[np.lexsort((-sv, -kv))[:K]]  # key desc, insertion_seq desc
            if sel.size >= MIN_MATCHES:
                L = self.lens[sel]
                b = (np.minimum(L, MAX_LEN) - 1) // w
                Lf = L.astype(np.float64)
                cnt = np.bincount(b, minlength=NBINS)
                s1 = np.bincount(b, weights=Lf, minlength=NBINS)
                s2 = np.bincount(b, weights=Lf * Lf, minlength=NBINS)
            else:
                cnt, s1, s2 = (x.astype(np.float64) for x in self.fb)
            nz = np.flatnonzero(cnt)
            sup = (s2[nz] + 2.0 * self.I[i] * s1[nz]) * 0.5 / cnt[nz]
            mas = cnt[nz] / cnt[nz].sum()
            G[i] = self.RK.gittins_min(sup, mas) if self.RK else O.gittins_min(sup, mas)
        return np.lexsort((self.ids, G))


def _cpu_sample(config: str) -> int:
    return 128 if config == "c2" else 16


def cpu_baseline(config: str, budget_s: float = 20.0):
    r = CpuRound(config, _cpu_sample(config))
    r.step()  # warm (BLAS threads, numba JIT)
    ts = []
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < budget_s and len(ts) < 5:
        t0 = time.perf_counter()
        r.step()
        ts.append(time.perf_counter() - t0)
    t = float(np.median(ts))
    return {"value": round(r.sample / t, 2), "unit": "requests/s", "cores": _NCPU, "kind": "port",
            "sample": (f"per step {r.sample} of the round's {CONFIGS[config]['nq']} queries scored "
                       f"against the whole {r.n}-row bank (no extrapolation), full stages 1-4; "
                       f"median of {len(ts)} steps; Gittins = reference servesim gittins_min "
                       f"({'numba, baseline/_ref' if r.RK else 'unavailable -> oracle'}); "
                       "similarity/top-k/histogram are SPEC-only (numpy restatement)")}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    config = "c4" if world > 1 else args.config
    r = CpuRound(config, _cpu_sample(config))
    for _ in range(max(1, args.warmup)):
        r.step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r.step()
    t = time.perf_counter() - t0
    value = r.sample * args.steps / t
    C = CONFIGS[config]
    cb = {"value": round(value, 2), "unit": "requests/s", "cores": _NCPU,
          "kind": "reference" if r.RK else "port",
          "sample": f"per step {r.sample} of the round's {C['nq']} queries x the whole "
                    f"{C['n_bank']}-row bank (no extrapolation)"}
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 2), "unit": "requests/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(1e3 * t / args.steps, 2), "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32/f64",
            "data": "synthetic (seeded clustered int8-valued embeddings, lognormal lengths; numpy)",
            "config": {"workload": C["workload"], "bank_rows": C["n_bank"], "dim": DIM,
                       "nq": C["nq"], "k": K, "nbins": NBINS, "theta": THETA,
                       "min_matches": MIN_MATCHES, "parallelism": f"host CPU, {_NCPU} threads"},
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
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-pure", action="store_true", help="skip the theta = -1 sub-record")
    ap.add_argument("--no-c4", action="store_true", help="skip the c4-on-one-GPU sub-record")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    ap.add_argument("--config", default=None, choices=["c2", "c3", "c4", "c5"],
                    help="c2 = headline at N = 1 (BASELINE configs[1]); c4 = 16M x 8192 "
                         "(default at N > 1); c3 = refresh storm; c5 = rolling replay")
    ap.add_argument("--sharded", action="store_true",
                    help="run the multi-GPU single-owner round even at N = 1")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="torch.distributed backend of the sharded round (gloo: a functional check "
                         "of the multi-rank path with several ranks sharing one GPU; not a measurement)")
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "p2p"],
                    help="candidate exchange of the sharded round")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.config is None:
        args.config = "c4" if (world > 1 or args.gpus > 1) else "c2"
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "c3":
        return run_c3(args)
    if args.config == "c5":
        return run_c5(args)
    run_ours(args)


if __name__ == "__main__":
    main()

"""TMEM read-back bandwidth and its interference with the int8 MMA
(tools/mma_peak.cu mma_peak_run2): drain alone, MMA alone, both at once."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _build  # noqa: E402

_build.build_probes()
lib = ctypes.CDLL(os.path.join(_build.TOOLS_DIR, "libmmapeak.so"))
lib.mma_peak_run2.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream()
CLK = 1.965e9


def run(tiles, n, dw, di):
    lib.mma_peak_run2(sms, min(tiles, 20), n, 1, dw, min(di, 2), ctypes.c_void_p(st.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0.record()
        rc = lib.mma_peak_run2(sms, tiles, n, 1, dw, di, ctypes.c_void_p(st.cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        best = min(best, e0.elapsed_time(e1))
    return best


for n in () if os.environ.get('NO_DRAIN') else (208, 256):
    nacc = 2 if 2 * n + 96 <= 512 else 1
    tiles = 6000
    t_mma = run(tiles, n, 0, 0)
    for dw in (4, 8):
        # drain bytes per pass over the accumulators: 128 lanes x nacc*n cols x 4 B (each
        # group of 4 warps covers all 128 lanes once)
        per_pass = 128 * (nacc * n // 32 * 32) * 4 * (dw // 4)
        iters = 2000
        t_dr = run(0, n, dw, iters)
        bw = per_pass * iters / (t_dr * 1e-3) / CLK  # bytes per clock per SM
        # drain sized to the same bytes per tile as the real kernel: one
        # accumulator (128 x n x 4 B) per tile
        di = max(1, tiles // nacc // (dw // 4))
        t_both = run(tiles, n, dw, di)
        print(f"N={n} nacc={nacc} drain_warps={dw}: mma alone {t_mma:.3f} ms "
              f"({tiles * 12 * 1e-3 / t_mma * 0 + t_mma * 1e-3 * CLK / (tiles * 12):.1f} cyc/MMA); "
              f"drain alone {bw:.1f} B/clk/SM; both (one accumulator drained per tile) "
              f"{t_both:.3f} ms ({t_both * 1e-3 * CLK / (tiles * 12):.1f} cyc/MMA)", flush=True)

# MMA issue with per-K-block barrier traffic (mode bit 0: commit, bit 1: wait on a
# completed barrier + tcgen05 fence)
lib.mma_peak_run3.argtypes = [ctypes.c_int] * 7 + [ctypes.c_void_p]
for n in (208,):
    for mode in (0, 2, 4, 8, 16, 0):
        tiles = 3000
        lib.mma_peak_run3(sms, 20, n, 1, 0, 0, mode, ctypes.c_void_p(st.cuda_stream))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record()
            assert lib.mma_peak_run3(sms, tiles, n, 1, 0, 0, mode, ctypes.c_void_p(st.cuda_stream)) == 0
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        print(f"N={n} mode={mode}: {best * 1e-3 * CLK / (tiles * 12):.1f} cyc/MMA", flush=True)

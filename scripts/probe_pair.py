"""Single-CTA vs CTA-pair int8 TS MMA rate, alone and with shared-memory store
traffic from 4 / 8 extra warps (tools/mma_peak.cu mma_pair_run)."""
import ctypes
import os
import subprocess
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _build  # noqa: E402

_build.build_probes()
lib = ctypes.CDLL(os.path.join(_build.TOOLS_DIR, "libmmapeak.so"))
lib.mma_pair_run.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream()


def clk():
    return subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits"],
                          capture_output=True, text=True).stdout.strip()


def run(tiles, n, sw, si, pair):
    ncta = sms if not pair else sms // 2 * 2
    rc = lib.mma_pair_run(ncta, min(tiles, 10), n, sw, min(si, 10), pair, ctypes.c_void_p(st.cuda_stream))
    assert rc == 0, rc
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize()
        e0.record()
        lib.mma_pair_run(ncta, tiles, n, sw, si, pair, ctypes.c_void_p(st.cuda_stream))
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


tiles = 1500
for n in (208, 256):
    for pair in (0, 1):
        t = run(tiles, n, 0, 0, pair)
        ops = 2.0 * 128 * n * 384 * tiles * (sms // 2 * 2 if pair else sms) * (2 if pair else 1) / (2 if pair else 1)
        # per SM: 128 x n x 384 MACs per tile either way
        ops = 2.0 * 128 * n * 384 * tiles * (sms // 2 * 2 if pair else sms)
        line = f"N={n} {'pair' if pair else 'single'}: {t:.3f} ms {ops / t / 1e9:7.1f} TOPS"
        for sw in (4, 8):
            si = 4000
            ts = run(0, n, sw, si, pair)
            si2 = max(1, int(si * t / ts))  # store traffic lasting as long as the MMAs
            tb = run(tiles, n, sw, si2, pair)
            sbw = sw * 32 * 16 * 4 * si / (ts * 1e-3) / 1.965e9  # bytes per clock per SM (approx)
            line += f" | {sw} store warps ({sbw:.0f} B/clk alone): both {tb:.3f} ms"
        print(line, "clk", clk(), flush=True)

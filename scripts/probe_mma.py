"""int8 tcgen05 MMA rate vs N and A placement (tools/mma_peak.cu), this GPU."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _build  # noqa: E402

_build.build_probes()
lib = ctypes.CDLL(os.path.join(_build.TOOLS_DIR, "libmmapeak.so"))
lib.mma_peak_run.argtypes = [ctypes.c_int] * 4 + [ctypes.c_void_p]
sms = torch.cuda.get_device_properties(0).multi_processor_count
st = torch.cuda.current_stream()
for n in (64, 96, 128, 160, 192, 208, 224, 256):
    for ts in (0, 1):
        tiles = 24000 * 208 // n
        if lib.mma_peak_run(sms, 20, n, ts, ctypes.c_void_p(st.cuda_stream)):
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            torch.cuda.synchronize()
            e0.record()
            lib.mma_peak_run(sms, tiles, n, ts, ctypes.c_void_p(st.cuda_stream))
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        ops = 2.0 * 128 * n * 384 * tiles * sms
        cyc = best * 1e-3 * 1.965e9 / (tiles * 12)
        print(f"N={n:3d} {'TS' if ts else 'SS'}: {ops / best / 1e9:7.1f} TOPS  {cyc:6.1f} cycles/MMA @1.965GHz")

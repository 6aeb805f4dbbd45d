"""How long does issuing a tcgen05.mma take (is the issue queue shallow)?"""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_07917_b200 import _build  # noqa: E402

_build.build_probes()
lib = ctypes.CDLL(os.path.join(_build.TOOLS_DIR, "libmmapeak.so"))
lib.mma_issue_timing.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
out = torch.zeros(256, dtype=torch.int64, device="cuda")
for n in (208, 256):
    for count in (48, 96):
        for _ in range(2):
            assert lib.mma_issue_timing(count, n, ctypes.c_void_p(out.data_ptr()),
                                        ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
            torch.cuda.synchronize()
        t = out[: count + 1].cpu().tolist()
        print(f"N={n} count={count}: issue-return clocks {t[:16]} ... {t[count - 4:count]}; all done {t[count]}"
              f" -> {t[count] / count:.1f} cyc/MMA")

"""torch.profiler breakdown of the device-resident c5 replay round."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_07917_b200 import _lib  # noqa: E402
from paper_2603_07917_b200.history import HistoryWindow  # noqa: E402
from paper_2603_07917_b200.replay_device import DeviceReplay, DeviceTrace  # noqa: E402
from paper_2603_07917_b200.scheduler import RoundConfig  # noqa: E402
from paper_2603_07917_b200.synthetic import inv_norm_device, make_bank_device  # noqa: E402

_lib.load()
emb, lens, _ = make_bank_device(bench.N_BANK, 384, bench.N_CLUSTERS, 0)
win = HistoryWindow(bench.N_BANK, 384)
win.push(emb, lens)
del emb, lens
n_trace = 1024 * 80
te, tl, _ = make_bank_device(n_trace, 384, bench.N_CLUSTERS, 0, member_seed=1000)
g = torch.Generator(device="cuda")
g.manual_seed(7)
tr = DeviceTrace(te, inv_norm_device(te), torch.randint(1, 4097, (n_trace,), generator=g,
                 device="cuda", dtype=torch.int32), tl)
cfg = RoundConfig(k=64, theta=0.8, min_matches=20, max_len=2048, nbins=128)
dr = DeviceReplay(win, tr, cfg, 1024, 32, 8192, 65536)
for _ in range(20):
    dr.round()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        dr.round()
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25))
print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25))

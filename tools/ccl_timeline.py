"""Kernel timeline of one 65536^2 kk_cluster_histogram call (torch.profiler /
CUPTI, not serialised): each kernel / memset / copy with its start offset and
duration, and the idle gaps between them.  Usage: python tools/ccl_timeline.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
lat = kk.Lattice(65536, 65536, 0.5, 0.6, 5)
lat.sweep(20, s)
lat.cluster_histogram_raw(1, stream=s)
lat.sweep(1, s)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    lat.cluster_histogram_raw(1, stream=s)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
ev.sort(key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
last = t0
for e in ev:
    st, en = e.time_range.start, e.time_range.end
    print(f"{(st - t0) / 1e3:9.3f} ms  +{(st - last) / 1e3:7.3f} gap  {(en - st) / 1e3:8.3f} ms  {e.name[:60]}")
    last = max(last, en)
print(f"total {(last - t0) / 1e3:.3f} ms")

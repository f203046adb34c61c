"""Pass-kernel throughput on the BASELINE configs (CUDA events, warm).
Usage: python tools/throughput_configs.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
for name, Lx, Ly, R, om, n in [("configs[0] 64x64", 64, 64, 1, 0.5, 200),
                               ("configs[1] 400x400", 400, 400, 1, 0.6, 200),
                               ("configs[2] 4096x4096", 4096, 4096, 1, 0.6, 50),
                               ("configs[3] 1024 x 400x400 replicas", 400, 400, 1024, 0.6, 10),
                               ("configs[4] 65536x65536", 65536, 65536, 1, 0.6, 2)]:
    L = kk.Lattice(Lx, Ly, 0.5, om, 11, replicas=R, init=kk.KK_INIT_BLOCK)
    L.sweep(2, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    L.sweep(n, s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    L.cluster_histogram(1, stream=s)  # workspace allocation outside the timing
    torch.cuda.synchronize()
    c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    c0.record(s)
    L.cluster_histogram(1, stream=s)
    c1.record(s)
    torch.cuda.synchronize()
    print(f"{name}: {n} sweeps {ms:.2f} ms -> {n * Lx * Ly * R / ms / 1e6:.1f} G site-updates/s; "
          f"cluster histogram {c0.elapsed_time(c1):.2f} ms", flush=True)
    L.close()

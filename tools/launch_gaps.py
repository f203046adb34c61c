"""Gaps between back-to-back pass launches: sum of per-pass event times vs the
wall time of the same passes on the device.  Usage: python tools/launch_gaps.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.current_stream()
for L_ in (1024, 2048, 4096, 8192):
    L = kk.Lattice(L_, L_, 0.5, 0.6, 3, init=kk.KK_INIT_BLOCK)
    L.sweep(2, st)
    torch.cuda.synchronize()
    n = 200
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(n):
        L.run_pass(kk.REGION_ALL, None, None, st)
        L.pass_commit()
    b.record(st)
    torch.cuda.synchronize()
    total = a.elapsed_time(b)
    ev = []
    for _ in range(n):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        L.run_pass(kk.REGION_ALL, None, None, st)
        e1.record(st)
        L.pass_commit()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    inner = sum(x.elapsed_time(y) for x, y in ev)
    print(f"{L_}^2: {n} passes {total:.2f} ms back to back, {total / n * 1e3:.1f} us/pass; "
          f"per-pass event sum {inner / n * 1e3:.1f} us/pass", flush=True)
    L.close()

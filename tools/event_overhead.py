"""Does recording CUDA events around every pass (bench.py's live roofline
timing) slow the pass loop down?  Usage: python tools/event_overhead.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import distributed as D  # noqa: E402

torch.cuda.set_device(0)
st = torch.cuda.current_stream()
sim = D.make_simulation(65536, 65536, 0.5, 0.6, 5, T=8, stream=st)
sim.sweep(2)
torch.cuda.synchronize()
for rep in range(3):
    for with_events in (False, True):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        ev = []
        a.record(st)
        for _ in range(100):
            if with_events:
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                sim.run_pass()
                e1.record(st)
                ev.append((e0, e1))
            else:
                sim.run_pass()
        b.record(st)
        torch.cuda.synchronize()
        tot = a.elapsed_time(b)
        inner = sum(x.elapsed_time(y) for x, y in ev) if ev else float("nan")
        print(f"events={with_events}: 100 passes {tot:.1f} ms (sum of per-pass {inner:.1f} ms)", flush=True)

"""Where the bench step's time goes (65536^2, 100 sweeps + observables + CCL).
Usage: python tools/step_breakdown.py [Lx] [rows] [sweeps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import distributed as D  # noqa: E402

Lx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
S = int(sys.argv[3]) if len(sys.argv) > 3 else 100
torch.cuda.set_device(0)
st = torch.cuda.current_stream()
sim = D.make_simulation(Lx, rows, 0.5, 0.6, 5, T=8, stream=st)
sim.sweep(2)
sim.observe(True)
torch.cuda.synchronize()


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record(st)
    return e


for rep in range(2):
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    a = ev()
    for _ in range(S * 2):
        sim.run_pass()
    b = ev()
    w1 = time.perf_counter()
    lat = sim.lat
    nab = lat.energy(stream=st)
    c = ev()
    na = lat.composition(stream=st)
    d = ev()
    s_ = lat.stats(True, stream=st)
    e = ev()
    torch.cuda.synchronize()
    w2 = time.perf_counter()
    h = lat.cluster_histogram(1, stream=st)
    f = ev()
    torch.cuda.synchronize()
    w3 = time.perf_counter()
    print(f"sweeps {a.elapsed_time(b):.1f} ms (host enqueue {1e3 * (w1 - w0):.1f} ms) | energy {b.elapsed_time(c):.2f}"
          f" | composition {c.elapsed_time(d):.2f} | stats {d.elapsed_time(e):.2f} | observables wall "
          f"{1e3 * (w2 - w1):.1f} | cluster histogram device {e.elapsed_time(f):.1f} ms wall {1e3 * (w3 - w2):.1f} ms"
          f" ({len(h[0])} distinct sizes) | total device {a.elapsed_time(f):.1f} ms", flush=True)

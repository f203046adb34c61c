"""Planar vs row-major tile kernel: site-updates/s per lattice (CUDA events,
random start equilibrated for a few sweeps), optionally with forced tiles.

  python tools/planar_rate.py [Lx ...]     env: KK_TWI / KK_THI / KK_PASS_THREADS apply to both
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402

torch.cuda.set_device(0)
s = torch.cuda.current_stream()
sizes = [int(a) for a in sys.argv[1:]] or [1024, 2048, 4096, 8192, 16384, 65536]
for Lx in sizes:
    for planar in ((1,) if os.environ.get('KK_ONLY_PLANAR') else (1, 0)):
        os.environ["KK_PLANAR"] = str(planar)
        os.environ.setdefault("KK_RESIDENT", "0")
        os.environ.setdefault("KK_CLUSTER", "0")
        os.environ.setdefault("KK_BAND", "0")
        L = kk.Lattice(Lx, Lx, 0.5, 0.6, 3)
        pl = kk.plan(Lx, Lx, n_sm=0)
        L.sweep(2, s)
        torch.cuda.synchronize()
        n = max(2, int(1.5e11 / (Lx * Lx)) // 2 * 2)
        n = min(n, 2000)
        best = 0.0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            L.sweep(n, s)
            e1.record(s)
            torch.cuda.synchronize()
            best = max(best, n * Lx * Lx / e0.elapsed_time(e1) / 1e6)
        st = L.stats()[0]
        print(f"{Lx}^2 {pl['kernel']:7s} TWI={pl['tile_words']} THI={pl['tile_rows']} nt={pl['threads']} "
              f"ctas={pl['ctas']} pdl={pl['pass_pdl']}: {best:8.1f} G/s  "
              f"(trivial {st[1] / st[0]:.3f}, accepted {st[2] / st[0]:.4f})", flush=True)
        L.close()

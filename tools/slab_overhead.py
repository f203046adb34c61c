"""Cost of the N>1 pass structure on one GPU: a 65536-row slab of a 2-slab
torus run through SlabDriver's split path (pack halos, interior bands on a
side stream, boundary bands on the main stream after the "exchange"), with
the exchange replaced by two device copies (send_top -> recv_bot, send_bot ->
recv_top), against the same lattice size through the plain single-GPU path.
The difference is what the slab decomposition itself costs per rank (NCCL
transfer time excluded; it overlaps the interior bands).
Usage: python tools/slab_overhead.py [Lx rows sweeps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1309_4349_b200 import kk  # noqa: E402
from paper_1309_4349_b200 import distributed as D  # noqa: E402


class CopyComm:
    """Stands in for TorchComm.exchange_*: the halos a periodic neighbour would send."""

    def __init__(self, stream):
        self.stream = stream

    def exchange_start(self, send_top, send_bot, recv_top, recv_bot):
        with torch.cuda.stream(self.stream):
            recv_bot.copy_(send_top)
            recv_top.copy_(send_bot)
        return []

    @staticmethod
    def exchange_wait(works):
        pass


def rate(drv, lat, sweeps, T, stream):
    drv.sweep(1, T)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    drv.sweep(sweeps, T)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    return sweeps * lat.Lx * lat.rows / (ms / 1e3) / 1e9, ms / (sweeps * 16 // T)


def main():
    Lx = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
    rows = int(sys.argv[2]) if len(sys.argv) > 2 else 65536
    sweeps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    T = 8
    torch.cuda.set_device(0)
    stream = torch.cuda.current_stream()
    dev = torch.device("cuda", 0)
    for rep in range(2):
        lat1 = kk.Lattice(Lx, rows, 0.5, 0.6, 7, iters_per_pass=T, init=kk.KK_INIT_BLOCK)
        drv1 = D.SlabDriver(D.GpuSlab(lat1, dev), None, 0, 1, stream)
        g1, p1 = rate(drv1, lat1, sweeps, T, stream)
        lat1.close()
        lat2 = kk.Lattice(Lx, 2 * rows, 0.5, 0.6, 7, iters_per_pass=T, init=kk.KK_INIT_BLOCK,
                          y_begin=0, y_count=rows)
        side = torch.cuda.Stream(device=dev)
        drv2 = D.SlabDriver(D.GpuSlab(lat2, dev), CopyComm(stream), 0, 2, stream, side)
        g2, p2 = rate(drv2, lat2, sweeps, T, stream)
        lat2.close()
        print(f"{Lx}x{rows}: plain {g1:.1f} G/s ({p1 * 1e3:.0f} us/pass), slab split {g2:.1f} G/s "
              f"({p2 * 1e3:.0f} us/pass): {100 * (1 - g2 / g1):+.2f}% per rank", flush=True)


if __name__ == "__main__":
    main()

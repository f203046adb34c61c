"""Row-slab multi-GPU driver (north_star: "Large lattices are slab-partitioned by
rows across the 8 GPUs of one box, with per-phase halo-row exchange via NCCL
over NVLink overlapped with interior updates").

One process per GPU.  Rank r holds global rows [r*rows, (r+1)*rows) of a
Lx x (rows*world) periodic lattice.  Every pass (T MPKK iterations, DESIGN.md
R8) needs hy = 3T rows above and below the slab as they were at the start of
the pass, so per pass:

    pack_halo (rows [0,hy) and [rows-hy,rows) of the current buffer)
    exchange  (send top -> previous rank's bottom halo, bottom -> next rank's top halo)
    interior bands   on a side stream, concurrently with the exchange
    boundary bands   after the exchange, reading the received halos
    commit           (flip buffers, advance the (sweep, iteration) counter)

Random numbers are keyed by global coordinates (R6), so the result is
bit-identical to a single-GPU run of the whole lattice for any world size.

The driver is backend-agnostic: ``GpuSlab`` adapts ``kk.Lattice`` (CUDA,
device halo buffers, NCCL); tests plug in a CPU backend and a gloo group to
check the decomposition logic on CPU.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import kk


# ----------------------------------------------------------------------- comm
class TorchComm:
    """torch.distributed plumbing: sums, gathers and the halo exchange.

    With NCCL (the product configuration) device tensors move directly.  With
    gloo and CUDA tensors (functional multi-rank tests on a single GPU, where
    NCCL refuses two ranks per device) they are staged through host memory."""

    TAG_DOWN, TAG_UP = 11, 12

    def __init__(self, rank: int, world: int, device=None, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.rank, self.world, self.group = rank, world, group
        self.device = device if device is not None else torch.device("cpu")
        self.stage = False
        if world > 1 and self.device.type == "cuda":
            self.stage = dist.get_backend(group) == "gloo"
        self.coll_device = torch.device("cpu") if self.stage else self.device

    def all_reduce_sum(self, a: np.ndarray) -> np.ndarray:
        if self.world == 1:
            return a
        t = self.torch.from_numpy(np.ascontiguousarray(a, np.int64)).to(self.coll_device)
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def all_gather_rows(self, a: np.ndarray) -> np.ndarray:
        """Concatenate a (n_i, k) int64 array from every rank (n_i may differ)."""
        if self.world == 1:
            return a
        torch = self.torch
        n = torch.tensor([a.shape[0]], dtype=torch.int64, device=self.coll_device)
        ns = [torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        m = max(int(x.item()) for x in ns)
        k = a.shape[1]
        pad = np.zeros((max(m, 1), k), np.int64)
        pad[: a.shape[0]] = a
        t = torch.from_numpy(pad).to(self.coll_device)
        outs = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return np.concatenate([o.cpu().numpy()[: int(c.item())] for o, c in zip(outs, ns)], axis=0)

    def all_gather_tensor(self, t):
        if self.world == 1:
            return [t]
        src = t.cpu() if self.stage else t
        outs = [self.torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(outs, src, group=self.group)
        return [o.to(t.device) for o in outs] if self.stage else outs

    def exchange_start(self, send_top, send_bot, recv_top, recv_bot):
        """send_top -> rank-1 (its bottom halo); send_bot -> rank+1 (its top halo)."""
        dist = self.dist
        prev = (self.rank - 1) % self.world
        nxt = (self.rank + 1) % self.world
        if self.stage:
            st, sb = send_top.cpu(), send_bot.cpu()
            rt, rb = self.torch.empty_like(st), self.torch.empty_like(sb)
            ops = [dist.P2POp(dist.isend, st, prev, self.group, self.TAG_DOWN),
                   dist.P2POp(dist.irecv, rb, nxt, self.group, self.TAG_DOWN),
                   dist.P2POp(dist.isend, sb, nxt, self.group, self.TAG_UP),
                   dist.P2POp(dist.irecv, rt, prev, self.group, self.TAG_UP)]
            return [_StagedRecv(dist.batch_isend_irecv(ops), [(rt, recv_top), (rb, recv_bot)])]
        ops = [dist.P2POp(dist.isend, send_top, prev, self.group, self.TAG_DOWN),
               dist.P2POp(dist.irecv, recv_bot, nxt, self.group, self.TAG_DOWN),
               dist.P2POp(dist.isend, send_bot, nxt, self.group, self.TAG_UP),
               dist.P2POp(dist.irecv, recv_top, prev, self.group, self.TAG_UP)]
        return dist.batch_isend_irecv(ops)

    @staticmethod
    def exchange_wait(works):
        for w in works:
            w.wait()


class _StagedRecv:
    """Host-staged exchange: wait for the host receives, then copy to device."""

    def __init__(self, works, copies):
        self.works, self.copies = works, copies

    def wait(self):
        for w in self.works:
            w.wait()
        for host, dev in self.copies:
            dev.copy_(host)


# -------------------------------------------------------------- GPU backend
class GpuSlab:
    """kk.Lattice + device halo buffers (torch tensors, so NCCL can move them)."""

    def __init__(self, lat: kk.Lattice, device):
        import torch
        self.lat = lat
        self.torch = torch
        self.device = device
        self.hy = lat.halo_rows
        self.replicas = lat.replicas
        self.Lx = lat.Lx

    def alloc_halo(self):
        return self.torch.zeros(self.replicas * self.hy * self.lat.W, dtype=self.torch.int32,
                                device=self.device)

    def pack_halo(self, top, bot, stream):
        self.lat.pack_halo(top.data_ptr(), bot.data_ptr(), stream)

    def run_pass(self, region, halo_top, halo_bot, stream):
        self.lat.run_pass(region, None if halo_top is None else halo_top.data_ptr(),
                          None if halo_bot is None else halo_bot.data_ptr(), stream)

    def commit(self):
        self.lat.pass_commit()

    def energy(self, halo_bot, stream):
        return self.lat.energy(None if halo_bot is None else halo_bot.data_ptr(), stream)[0]

    def composition(self, stream):
        return self.lat.composition(stream)

    def stats(self, reset, stream):
        return self.lat.stats(reset, stream)

    def cluster_histogram_rows(self, target, stream):
        """Full periodic lattice: [(size, count)] of replica 0."""
        return self.lat.cluster_histogram(target, stream=stream)[0]

    def cluster_histogram_array(self, target, stream):
        """As cluster_histogram_rows, as an (n, 2) int64 array (no per-row Python objects)."""
        return self.lat.cluster_histogram_raw(target, stream=stream)[:, 1:]

    # slab cluster histogram (multi-GPU)
    def alloc_cluster_buffers(self):
        t = self.torch
        Lx = self.lat.Lx
        cap = 2 * Lx + 16
        return (t.empty(Lx, dtype=t.int32, device=self.device), t.empty(Lx, dtype=t.int32, device=self.device),
                t.empty(cap, dtype=t.int64, device=self.device), cap)

    def cluster_slab(self, target, bufs, stream):
        top, bot, sizes, cap = bufs
        return self.lat.cluster_slab(target, top.data_ptr(), bot.data_ptr(), sizes.data_ptr(), cap, stream)

    def cluster_join(self, Lx, nslabs, top_all, bot_all, offsets, sizes_all, n_nodes, stream):
        return kk.cluster_join(Lx, nslabs, top_all.data_ptr(), bot_all.data_ptr(), offsets,
                               sizes_all.data_ptr(), n_nodes, stream)

    def close(self):
        self.lat.close()


# ------------------------------------------------------------- random start
def distributed_random_init(lat, comm, fraction_A: float, Lx: int, Ly: int):
    """Exact-composition random start (R7) over all slabs: histograms summed
    and ties gathered here; the bin choice and the tie cut are the library's
    host steps (kk_init_select_choose / kk_init_select_cut)."""
    R = lat.replicas
    nA = int(np.floor(fraction_A * Lx * Ly + 0.5))
    need = np.full(R, nA, np.int64)
    prefix = np.zeros(R, np.uint32)
    for level in range(3):
        h = lat.select_hist(level, None if level == 0 else prefix)
        h = comm.all_reduce_sum(h)
        kk.select_choose(level, h, need, prefix)
    ties = comm.all_gather_rows(lat.select_ties(prefix))
    lat.select_apply(prefix, kk.select_cut(ties, R, need))


# ------------------------------------------------------------------ driver
class SlabDriver:
    def __init__(self, backend, comm: Optional[TorchComm], rank: int, world: int,
                 stream=None, side_stream=None):
        self.be, self.comm, self.rank, self.world = backend, comm, rank, world
        self.stream, self.side = stream, side_stream
        if world > 1:
            self.send_top, self.send_bot = backend.alloc_halo(), backend.alloc_halo()
            self.recv_top, self.recv_bot = backend.alloc_halo(), backend.alloc_halo()

    def run_pass(self):
        be = self.be
        if self.world == 1:
            be.run_pass(kk.REGION_ALL, None, None, self.stream)
            be.commit()
            return
        be.pack_halo(self.send_top, self.send_bot, self.stream)
        with self._on_stream():
            # NCCL orders its send after the current stream (the halo pack) and
            # Work.wait() orders the current stream after the receive, so both
            # happen with the driver's stream current: the boundary pass below
            # runs on that stream
            works = self.comm.exchange_start(self.send_top, self.send_bot, self.recv_top, self.recv_bot)
        if self.side is not None:
            self.side.wait_stream(self.stream)
            be.run_pass(kk.REGION_INTERIOR, None, None, self.side)
        else:
            be.run_pass(kk.REGION_INTERIOR, None, None, self.stream)
        with self._on_stream():
            self.comm.exchange_wait(works)
        be.run_pass(kk.REGION_BOUNDARY, self.recv_top, self.recv_bot, self.stream)
        if self.side is not None:
            self.stream.wait_stream(self.side)
        be.commit()

    def _on_stream(self):
        """Context making the driver's CUDA stream current (no-op without one)."""
        import contextlib
        if self.stream is None or not hasattr(self.stream, "cuda_stream"):
            return contextlib.nullcontext()
        import torch
        return torch.cuda.stream(self.stream)

    def sweep(self, n: int, T: int):
        for _ in range(n * (16 // T)):
            self.run_pass()

    def refresh_halos(self):
        if self.world > 1:
            self.be.pack_halo(self.send_top, self.send_bot, self.stream)
            with self._on_stream():
                self.comm.exchange_wait(self.comm.exchange_start(self.send_top, self.send_bot,
                                                                 self.recv_top, self.recv_bot))

    def cluster_histogram(self, target: int = 1):
        """Cluster-size histogram [(size, count)] of the whole lattice (R9), on
        rank 0 (None elsewhere).  Multi-GPU: slab-local labelling, open clusters
        (touching a slab's first/last row) joined across slab boundaries on
        rank 0."""
        be = self.be
        if self.world == 1:
            return be.cluster_histogram_rows(target, self.stream)
        if not hasattr(self, "_cbufs"):
            self._cbufs = be.alloc_cluster_buffers()
        rows, n_open = be.cluster_slab(target, self._cbufs, self.stream)
        ns = self.comm.all_gather_rows(np.array([[n_open]], np.int64))[:, 0]
        all_rows = self.comm.all_gather_rows(np.asarray(rows, np.int64).reshape(-1, 2))
        tops = self.comm.all_gather_tensor(self._cbufs[0])
        bots = self.comm.all_gather_tensor(self._cbufs[1])
        sizes = self.comm.all_gather_tensor(self._cbufs[2])
        if self.rank != 0:
            return None
        torch = self.comm.torch
        offsets = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
        sizes_all = torch.cat([sz[: int(n)] for sz, n in zip(sizes, ns)]) if int(ns.sum()) else sizes[0][:1]
        jrows = be.cluster_join(be.Lx, self.world, torch.cat(tops), torch.cat(bots), offsets, sizes_all,
                                int(ns.sum()), self.stream)
        return kk.hist_merge(np.concatenate([np.asarray(all_rows, np.int64).reshape(-1, 2),
                                             np.asarray(jrows, np.int64).reshape(-1, 2)]))

    def observe(self, ccl: bool = True) -> dict:
        """N_AB, composition and counters summed over slabs, and the cluster
        histogram of the A sites (R9)."""
        self.refresh_halos()
        nab = np.asarray(self.be.energy(self.recv_bot if self.world > 1 else None, self.stream), np.int64)
        na = np.asarray(self.be.composition(self.stream), np.int64)
        st = np.asarray(self.be.stats(True, self.stream), np.int64)
        if self.world > 1:
            nab = self.comm.all_reduce_sum(nab)
            na = self.comm.all_reduce_sum(na)
            st = self.comm.all_reduce_sum(st)
        out = {"n_ab": nab.tolist(), "n_a": na.tolist(), "attempted": st[:, 0].tolist(),
               "trivial": st[:, 1].tolist(), "accepted": st[:, 2].tolist(), "dnab_sum": st[:, 3].tolist()}
        if ccl:
            h = (self.be.cluster_histogram_array(1, self.stream) if self.world == 1 and
                 hasattr(self.be, "cluster_histogram_array") else self.cluster_histogram(1))
            if h is not None:
                h = np.asarray(h, np.int64).reshape(-1, 2)
                out["clusters_A"] = int(h[:, 1].sum())
                out["largest_A"] = int(h[:, 0].max()) if len(h) else 0
        return out


class Simulation:
    """What bench.py drives: a full lattice (1 GPU) or one slab of it."""

    def __init__(self, driver: SlabDriver, lat: kk.Lattice, T: int):
        self.driver, self.lat, self.T = driver, lat, T

    def run_pass(self):
        self.driver.run_pass()

    def sweep(self, n: int):
        self.driver.sweep(n, self.T)

    def observe(self, ccl=True):
        return self.driver.observe(ccl)

    def packed_words(self) -> int:
        return self.lat.replicas * self.lat.rows * self.lat.W

    def upload_packed(self, host_ptr: int):
        self.lat.set_packed_ptr(host_ptr, self.driver.stream)

    # double-buffered host I/O through the C ABI (kk_upload_packed_async ...)
    def upload_async(self, host_ptr: int, copy_stream):
        self.lat.upload_async(host_ptr, copy_stream)

    def commit_upload(self, stream=None):
        self.lat.commit_upload(stream if stream is not None else self.driver.stream)

    def snapshot(self, stream=None):
        self.lat.snapshot(stream if stream is not None else self.driver.stream)

    def download_async(self, host_ptr: int, copy_stream):
        self.lat.download_async(host_ptr, copy_stream)

    def upload_device(self, dev_ptr: int, stream=None):
        """Lattice <- packed words at a device address (same layout)."""
        self.lat.copy_packed_device(dev_ptr, True, stream if stream is not None else self.driver.stream)

    def download_device(self, dev_ptr: int, stream=None):
        """Packed words of the lattice -> a device address."""
        self.lat.copy_packed_device(dev_ptr, False, stream if stream is not None else self.driver.stream)

    def download_packed(self, host_ptr: int):
        import ctypes
        kk._check(kk.load().kk_get_lattice_packed(self.lat.handle, ctypes.c_void_p(host_ptr),
                                                  kk.stream_ptr(self.driver.stream)),
                  "kk_get_lattice_packed")

    def close(self):
        self.lat.close()


def slab_rows(Ly: int, world: int) -> int:
    """Rows per rank of a row-slab split: every rank holds the same number of
    rows, a multiple of 4 (the centre classes, R10); anything else would leave
    rows unsimulated or break the phase of the slabs below."""
    if world < 1 or Ly % world != 0 or (Ly // world) % 4 != 0:
        raise ValueError(f"Ly={Ly} does not split into {world} slabs of equal height divisible by 4")
    return Ly // world


def make_simulation(Lx: int, Ly: int, fraction_A: float, omega: float, seed: int, T: int = 4,
                    world: int = 1, rank: int = 0, device: int = 0, stream=None) -> Simulation:
    import torch
    if world == 1:
        lat = kk.Lattice(Lx, Ly, fraction_A, omega, seed, iters_per_pass=T, device=device)
        drv = SlabDriver(GpuSlab(lat, torch.device("cuda", device)), None, 0, 1, stream)
        return Simulation(drv, lat, T)
    rows = slab_rows(Ly, world)
    lat = kk.Lattice(Lx, Ly, fraction_A, omega, seed, init=kk.KK_INIT_EMPTY, iters_per_pass=T,
                     y_begin=rank * rows, y_count=rows, device=device)
    comm = TorchComm(rank, world, torch.device("cuda", device))
    distributed_random_init(lat, comm, fraction_A, Lx, Ly)
    side = torch.cuda.Stream(device=device)
    drv = SlabDriver(GpuSlab(lat, torch.device("cuda", device)), comm, rank, world, stream, side)
    return Simulation(drv, lat, T)

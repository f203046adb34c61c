"""Multi-process (gloo, world_size 2 and 4) checks of the row-slab driver on CPU.

The product driver (paper_1309_4349_b200/distributed.py: halo packing,
exchange directions/tags, interior/boundary split, distributed random start,
observable reductions) runs unchanged; only the per-slab compute backend is a
CPU stand-in built from the oracle (test infrastructure).  The gathered result
must equal the oracle on the whole lattice bit-exactly.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O

NB_FWD = [(1, 0), (0, 1), (1, 1)]


class OracleSlab:
    """CPU stand-in with the GpuSlab interface (uint8 rows, int32 halos)."""

    def __init__(self, Lx, Ly, rows, y_begin, omega, seed, T, start):
        self.Lx, self.Ly, self.rows, self.y0 = Lx, Ly, rows, y_begin
        self.omega, self.seed, self.T, self.hy = omega, seed, T, 3 * T
        self.cur = start.copy()
        self.nxt = start.copy()
        self.sweep, self.j = 0, 0
        self.st = np.zeros((1, 4), np.int64)
        self.replicas = 1
        self.Lx = Lx

    # --- pass protocol
    def alloc_halo(self):
        return torch.zeros(self.hy * self.Lx, dtype=torch.int32)

    def pack_halo(self, top, bot, stream):
        top.copy_(torch.from_numpy(self.cur[: self.hy].astype(np.int32).reshape(-1)))
        bot.copy_(torch.from_numpy(self.cur[self.rows - self.hy:].astype(np.int32).reshape(-1)))

    def _window(self, win, y_origin, r0, r1):
        st = O.window_iterations(win, self.Ly, y_origin, self.omega, self.seed, self.sweep, 0,
                                 self.j, self.T, r0, r1)
        self.st += np.array([[st["attempted"], st["trivial"], st["accepted"], st["dnab_sum"]]])
        return win

    def run_pass(self, region, halo_top, halo_bot, stream):
        hy, rows = self.hy, self.rows
        if region == 1:    # interior rows [hy, rows-hy): local data only
            if rows > 2 * hy:
                win = self.cur.copy()
                self._window(win, self.y0, hy, rows - hy)
                self.nxt[hy:rows - hy] = win[hy:rows - hy]
        elif region == 2:  # boundary rows [0,hy) and [rows-hy,rows): need the halos
            top = halo_top.numpy().reshape(hy, self.Lx).astype(np.uint8)
            bot = halo_bot.numpy().reshape(hy, self.Lx).astype(np.uint8)
            pad = np.concatenate([top, self.cur, bot])
            if rows > 2 * hy:
                w1 = pad.copy()
                self._window(w1, self.y0 - hy, hy, 2 * hy)
                w2 = pad.copy()
                self._window(w2, self.y0 - hy, rows, rows + hy)
                self.nxt[:hy] = w1[hy:2 * hy]
                self.nxt[rows - hy:] = w2[rows:rows + hy]
            else:
                w = pad.copy()
                self._window(w, self.y0 - hy, hy, hy + rows)
                self.nxt[:] = w[hy:hy + rows]

    def commit(self):
        self.cur, self.nxt = self.nxt, self.cur.copy()
        self.j += self.T
        if self.j == 16:
            self.j = 0
            self.sweep += 1

    # --- observables
    def energy(self, halo_bot, stream):
        lat = self.cur
        up = np.concatenate([lat[1:], halo_bot.numpy().reshape(self.hy, self.Lx)[:1].astype(np.uint8)])
        n = int((lat != np.roll(lat, -1, 1)).sum())
        n += int((lat != up).sum()) + int((lat != np.roll(up, -1, 1)).sum())
        return np.array([n])

    def composition(self, stream):
        return np.array([int(self.cur.sum())])

    def stats(self, reset, stream):
        s = self.st.copy()
        if reset:
            self.st[:] = 0
        return s

    # --- slab cluster histogram (same contract as kk_cluster_slab / kk_cluster_join)
    def alloc_cluster_buffers(self):
        cap = 2 * self.Lx + 16
        return (torch.zeros(self.Lx, dtype=torch.int32), torch.zeros(self.Lx, dtype=torch.int32),
                torch.zeros(cap, dtype=torch.int64), cap)

    def cluster_slab(self, target, bufs, stream):
        top, bot, sizes, cap = bufs
        lat, rows, Lx = self.cur, self.rows, self.Lx
        lab = -np.ones((rows, Lx), np.int64)
        comps = []
        for y0 in range(rows):
            for x0 in range(Lx):
                if lat[y0, x0] != target or lab[y0, x0] >= 0:
                    continue
                stack, n, open_ = [(y0, x0)], 0, False
                lab[y0, x0] = len(comps)
                while stack:
                    y, x = stack.pop()
                    n += 1
                    open_ |= (y == 0 or y == rows - 1)
                    for dx, dy in [(1, 0), (1, 1), (0, 1), (-1, 0), (-1, -1), (0, -1)]:
                        yy, xx = y + dy, (x + dx) % Lx
                        if 0 <= yy < rows and lat[yy, xx] == target and lab[yy, xx] < 0:
                            lab[yy, xx] = len(comps)
                            stack.append((yy, xx))
                comps.append((n, open_))
        open_ids, complete = {}, {}
        for c, (n, o) in enumerate(comps):
            if o:
                open_ids[c] = len(open_ids)
                sizes[open_ids[c]] = n
            else:
                complete[n] = complete.get(n, 0) + 1
        none = -1  # 0xFFFFFFFF as int32
        top.copy_(torch.tensor([open_ids[l] if l >= 0 else none for l in lab[0]], dtype=torch.int32))
        bot.copy_(torch.tensor([open_ids[l] if l >= 0 else none for l in lab[rows - 1]], dtype=torch.int32))
        return np.array(sorted(complete.items()), np.int64).reshape(-1, 2), len(open_ids)

    def cluster_join(self, Lx, nslabs, top_all, bot_all, offsets, sizes_all, n_nodes, stream):
        par = list(range(n_nodes))

        def find(a):
            while par[a] != a:
                a = par[a]
            return a
        top = top_all.numpy().reshape(nslabs, Lx)
        bot = bot_all.numpy().reshape(nslabs, Lx)
        for s in range(nslabs):
            sn = (s + 1) % nslabs
            for x in range(Lx):
                a = bot[s, x]
                if a < 0:
                    continue
                for b in (top[sn, x], top[sn, (x + 1) % Lx]):
                    if b >= 0:
                        ra, rb = find(a + offsets[s]), find(b + offsets[sn])
                        if ra != rb:
                            par[max(ra, rb)] = min(ra, rb)
        tot = {}
        sz = sizes_all.numpy()
        for i in range(n_nodes):
            r = find(i)
            tot[r] = tot.get(r, 0) + int(sz[i])
        h = {}
        for v in tot.values():
            h[v] = h.get(v, 0) + 1
        return np.array(sorted(h.items()), np.int64).reshape(-1, 2)

    # --- distributed random start
    def _keys(self):
        k = np.zeros((self.rows, self.Lx), np.int64)
        for y in range(self.rows):
            for x in range(self.Lx):
                k[y, x] = O.philox4x32_10((x, self.y0 + y, 0, 0x20), (self.seed & 0xFFFFFFFF, self.seed >> 32))[0]
        return k

    def select_hist(self, level, prefix):
        k = self._keys().reshape(-1)
        h = np.zeros((1, 2048), np.int64)
        if level == 0:
            np.add.at(h[0], k >> 21, 1)
        elif level == 1:
            m = (k >> 21) == int(prefix[0])
            np.add.at(h[0], (k[m] >> 10) & 2047, 1)
        else:
            m = (k >> 10) == int(prefix[0])
            np.add.at(h[0], k[m] & 1023, 1)
        return h

    def select_ties(self, K):
        k = self._keys()
        ys, xs = np.nonzero(k == int(K[0]))
        return np.stack([np.zeros_like(ys), (self.y0 + ys) * self.Lx + xs], 1).astype(np.int64)

    def select_apply(self, K, cut):
        k = self._keys()
        y, x = np.mgrid[0:self.rows, 0:self.Lx]
        idx = (self.y0 + y) * self.Lx + x
        self.cur = ((k < int(K[0])) | ((k == int(K[0])) & (idx < int(cut[0])))).astype(np.uint8)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1309_4349_b200.distributed import SlabDriver, TorchComm, distributed_random_init
        Lx, Ly, T, omega, seed, n, f = cfg
        rows = Ly // world
        be = OracleSlab(Lx, Ly, rows, rank * rows, omega, seed, T, np.zeros((rows, Lx), np.uint8))
        comm = TorchComm(rank, world)
        distributed_random_init(be, comm, f, Lx, Ly)
        init = be.cur.copy()
        drv = SlabDriver(be, comm, rank, world)
        drv.sweep(n, T)
        obs = drv.observe(ccl=True)
        obs["hist"] = {t: drv.cluster_histogram(t) for t in (0, 1)}
        q.put((rank, init, be.cur.copy(), obs))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,Lx,Ly,T,n", [(2, 16, 48, 4, 3), (2, 8, 32, 2, 2), (4, 16, 96, 4, 2),
                                              (2, 24, 40, 1, 2),
                                              # strong scaling: one 16 x 96 lattice over 2, 4 and 8 ranks
                                              (2, 16, 96, 4, 1), (8, 16, 96, 4, 1)])
def test_slab_driver_matches_single_lattice(world, Lx, Ly, T, n):
    omega, seed, f = 0.7, 4321, 0.45
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, (Lx, Ly, T, omega, seed, n, f), q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    init = np.concatenate([r[1] for r in res])
    final = np.concatenate([r[2] for r in res])
    ref = O.init_random(Lx, Ly, f, seed)
    assert np.array_equal(init, ref)                     # distributed exact-composition start
    st = O.run(ref, omega, seed, n)
    assert np.array_equal(final, ref)                    # slabs + halos == whole lattice
    obs = res[0][3]
    assert obs["n_ab"] == [O.n_ab(ref)]
    assert obs["n_a"] == [int(ref.sum())]
    assert obs["attempted"] == [st["attempted"]] and obs["accepted"] == [st["accepted"]]
    assert obs["trivial"] == [st["trivial"]] and obs["dnab_sum"] == [st["dnab_sum"]]
    for t in (0, 1):                                     # slab-local labels + join == whole lattice
        assert [tuple(r) for r in obs["hist"][t]] == O.cluster_histogram(ref, t)
    assert obs["clusters_A"] == sum(c for _, c in O.cluster_histogram(ref, 1))
    for r in res[1:]:
        assert r[3]["hist"][1] is None                   # only rank 0 assembles the histogram


def test_slab_rows_rejects_uneven_splits():
    """make_simulation's split: equal slabs whose height is a multiple of 4
    (R10); anything else would leave rows unsimulated."""
    from paper_1309_4349_b200.distributed import slab_rows
    assert slab_rows(65536, 8) == 8192 and slab_rows(96, 8) == 12
    for Ly, world in [(1028, 8), (100, 3), (96, 16), (96, 0)]:
        with pytest.raises(ValueError):
            slab_rows(Ly, world)

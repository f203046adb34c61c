"""Slab kernels on ONE GPU: the multi-GPU data path emulated in one process.

S slab handles hold consecutive row bands of one lattice on the same device;
the halo exchange NCCL would do is done with device-to-device tensor copies
(no kernel ever waits on another).  Checks, bit-exact against the oracle on
the whole lattice: kk_pass with REGION_INTERIOR / REGION_BOUNDARY and
received halos, kk_pack_halo, slab energy with the next slab's first row,
counters, the distributed random start (kk_init_select_*), and the slab
cluster histogram + kk_cluster_join.
"""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_4349_b200 import build
    build.build()


def _slabs(Lx, Ly, S, omega, seed, T, init_full=None, random_init=False, f=0.5):
    import torch
    from paper_1309_4349_b200 import kk
    rows = Ly // S
    labs = [kk.Lattice(Lx, Ly, f, omega, seed, init=kk.KK_INIT_EMPTY, iters_per_pass=T,
                       y_begin=s * rows, y_count=rows) for s in range(S)]
    if random_init:
        # distributed exact-composition start: sum histograms over slabs; the
        # bin choice and the tie cut are the library's host steps
        nA = int(np.floor(f * Lx * Ly + 0.5))
        need = np.array([nA], np.int64)
        prefix = np.zeros(1, np.uint32)
        for level in range(3):
            h = sum(L.select_hist(level, None if level == 0 else prefix) for L in labs)
            kk.select_choose(level, h, need, prefix)
        ties = np.concatenate([L.select_ties(prefix) for L in labs])
        cut = kk.select_cut(ties, 1, need)
        for L in labs:
            L.select_apply(prefix, cut)
    else:
        for s, L in enumerate(labs):
            L.set_lattice(init_full[s * rows:(s + 1) * rows][None])
    dev = torch.device("cuda", torch.cuda.current_device())
    hy = labs[0].halo_rows
    mk = lambda: torch.zeros(hy * labs[0].W, dtype=torch.int32, device=dev)  # noqa: E731
    bufs = [dict(st=mk(), sb=mk(), rt=mk(), rb=mk()) for _ in range(S)]
    return labs, bufs


def _exchange(labs, bufs):
    S = len(labs)
    for L, b in zip(labs, bufs):
        L.pack_halo(b["st"].data_ptr(), b["sb"].data_ptr())
    for s in range(S):
        bufs[s]["rt"].copy_(bufs[(s - 1) % S]["sb"])   # rows above me = previous slab's bottom rows
        bufs[s]["rb"].copy_(bufs[(s + 1) % S]["st"])   # rows below me = next slab's top rows


def _run(labs, bufs, n_passes):
    from paper_1309_4349_b200 import kk
    for _ in range(n_passes):
        _exchange(labs, bufs)
        for L, b in zip(labs, bufs):
            L.run_pass(kk.REGION_INTERIOR, None, None)
            L.run_pass(kk.REGION_BOUNDARY, b["rt"].data_ptr(), b["rb"].data_ptr())
        for L in labs:
            L.pass_commit()


@pytest.mark.parametrize("Lx,Ly,S,T,n,planar", [(64, 96, 2, 4, 3, 0), (72, 120, 3, 8, 2, 0), (128, 64, 4, 2, 2, 0),
                                                (1024, 2048, 4, 8, 1, 0), (2048, 512, 2, 8, 2, 0),
                                                (128, 64, 4, 2, 2, 2), (1024, 2048, 4, 8, 1, 2),
                                                (2048, 512, 2, 8, 2, 2), (512, 384, 3, 4, 2, 2)])
def test_slab_passes_match_whole_lattice(Lx, Ly, S, T, n, planar):
    """Slab passes (halo pack, interior / boundary regions, halos received in
    the public row-major layout) equal the whole-lattice oracle; planar=2
    runs the planar tile kernel on the slabs (halo rows converted on staging,
    kk_pack_halo converting planar rows back)."""
    import os
    os.environ["KK_THI"] = "8"          # several bands per slab: interior + boundary regions both used
    os.environ["KK_PLANAR"] = str(planar)
    try:
        omega, seed = 0.7, 99
        full = O.init_random(Lx, Ly, 0.5, seed)
        labs, bufs = _slabs(Lx, Ly, S, omega, seed, T, init_full=full)
        from paper_1309_4349_b200 import kk
        assert kk.plan(Lx, Ly, y_begin=0, y_count=Ly // S, iters_per_pass=T)["kernel"] == (
            "planar" if planar else "tile")
    finally:
        os.environ.pop("KK_THI", None)
        os.environ.pop("KK_PLANAR", None)
    _run(labs, bufs, n * 16 // T)
    got = np.concatenate([L.get_lattice()[0] for L in labs])
    st = sum(L.stats()[0] for L in labs)
    ref = full.copy()
    ost = O.run(ref, omega, seed, n)
    assert np.array_equal(got, ref)
    assert list(st) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]
    _exchange(labs, bufs)
    nab = sum(int(L.energy(b["rb"].data_ptr())[0][0]) for L, b in zip(labs, bufs))
    assert nab == O.n_ab(ref)
    assert sum(int(L.composition()[0]) for L in labs) == int(ref.sum())


def test_distributed_random_start():
    labs, _ = _slabs(96, 64, 4, 0.5, 2024, 4, random_init=True, f=0.37)
    got = np.concatenate([L.get_lattice()[0] for L in labs])
    assert np.array_equal(got, O.init_random(96, 64, 0.37, 2024))


@pytest.mark.parametrize("Lx,Ly,S,f", [(64, 96, 2, 0.5), (520, 400, 4, 0.45), (256, 64, 1, 0.6),
                                       (1024, 256, 8, 0.55)])
def test_slab_cluster_histogram_join(Lx, Ly, S, f):
    import torch
    from paper_1309_4349_b200 import kk
    from tests import inputs
    full = inputs.random_lattice(Lx, Ly, f, seed=Lx + S)
    labs, _ = _slabs(Lx, Ly, S, 0.5, 1, 4, init_full=full)
    dev = torch.device("cuda", torch.cuda.current_device())
    for target in (0, 1):
        tops, bots, sizes, ns, hist = [], [], [], [], {}
        for L in labs:
            top = torch.empty(Lx, dtype=torch.int32, device=dev)
            bot = torch.empty(Lx, dtype=torch.int32, device=dev)
            sz = torch.empty(2 * Lx + 16, dtype=torch.int64, device=dev)
            rows, n_open = L.cluster_slab(target, top.data_ptr(), bot.data_ptr(), sz.data_ptr(), 2 * Lx + 16)
            for s_, c in rows.tolist():
                hist[s_] = hist.get(s_, 0) + c
            tops.append(top)
            bots.append(bot)
            sizes.append(sz[:n_open])
            ns.append(n_open)
        offsets = np.concatenate([[0], np.cumsum(ns)[:-1]]).astype(np.int64)
        sizes_all = torch.cat(sizes) if sum(ns) else torch.zeros(1, dtype=torch.int64, device=dev)
        top_all, bot_all = torch.cat(tops), torch.cat(bots)
        jrows = kk.cluster_join(Lx, S, top_all.data_ptr(), bot_all.data_ptr(), offsets, sizes_all.data_ptr(),
                                sum(ns))
        for s_, c in np.asarray(jrows).tolist():
            hist[s_] = hist.get(s_, 0) + c
        assert sorted(hist.items()) == O.cluster_histogram(full, target)

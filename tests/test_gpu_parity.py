"""Parity of the CUDA path (through the C ABI) with the oracle — bit-exact for
lattice state, N_AB, composition, counters and cluster histograms (north_star:
"GPU results must match the oracle bit-exactly").

Sizes span several tiles and ragged tails (KK_TWI / KK_THI force small tiles),
Lx % 32 != 0, all iterations-per-pass settings, replicas, and the BASELINE
workload sizes (64x64 x 1000 sweeps; 400x400; 4096x4096; the 65536x65536 bench
lattice via sampled window parity and invariants).
"""
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1309_4349_b200 import build
    build.build()


def _lat(*a, env=None, **k):
    from paper_1309_4349_b200 import kk
    old = {}
    for key, v in (env or {}).items():
        old[key] = os.environ.get(key)
        os.environ[key] = str(v)
    try:
        return kk.Lattice(*a, **k)
    finally:
        for key, v in old.items():
            if v is None:
                os.environ.pop(key, None)
            else:
                os.environ[key] = v


def _oracle_stats(st):
    return [st["attempted"], st["trivial"], st["accepted"], st["dnab_sum"]]


def test_acceptance_table_matches_oracle_rule():
    from paper_1309_4349_b200 import kk
    for om in [0.2, 0.5, 0.6, 1.0, -0.7, 0.0, 3.0]:
        L = _lat(8, 4, 0.5, om, 1)
        thr = L.acceptance_table()
        for v in range(-3, 4):
            dE = om * 2 * v
            t = int(thr[v + 3])
            assert O.metropolis_accept(dE, t)
            if t < 0xFFFFFFFF:
                assert not O.metropolis_accept(dE, t + 1)
        L.close()
    del kk


@pytest.mark.parametrize("Lx,Ly,f,R", [(8, 4, 0.5, 1), (40, 12, 0.3, 1), (64, 64, 0.5, 1),
                                       (72, 20, 0.7, 2), (400, 400, 0.3, 2), (1024, 36, 0.5, 1)])
def test_init_random_and_block_parity(Lx, Ly, f, R):
    from paper_1309_4349_b200 import kk
    seed = 1000 + Lx
    L = _lat(Lx, Ly, f, 0.5, seed, replicas=R)
    got = L.get_lattice()
    for r in range(R):
        assert np.array_equal(got[r], O.init_random(Lx, Ly, f, seed, replica=r))
    assert (L.composition() == O.count_a_for(Lx * Ly, f)).all()
    B = _lat(Lx, Ly, f, 0.5, seed, replicas=R, init=kk.KK_INIT_BLOCK)
    gb = B.get_lattice()
    for r in range(R):
        assert np.array_equal(gb[r], O.init_block(Lx, Ly, f))


def test_set_get_roundtrip_and_observables():
    for (Lx, Ly) in [(8, 4), (40, 12), (96, 8), (1000, 16)]:
        a = inputs.random_lattice(Lx, Ly, 0.4, seed=Lx)
        from paper_1309_4349_b200 import kk
        L = _lat(Lx, Ly, 0.5, 0.5, 3, init=kk.KK_INIT_EMPTY)
        L.set_lattice(a[None])
        assert np.array_equal(L.get_lattice()[0], a)
        nab, e = L.energy()
        assert nab[0] == O.n_ab(a)
        assert e[0] == 0.5 * O.n_ab(a)
        assert L.composition()[0] == int(a.sum())
        packed = L.get_packed()
        assert np.array_equal(inputs.unpack_rows(packed, Lx)[0], a)


def _run_parity(Lx, Ly, f, omega, seed, n, T=0, env=None, R=1, start=None):
    from paper_1309_4349_b200 import kk
    L = _lat(Lx, Ly, f, omega, seed, replicas=R, iters_per_pass=T, env=env,
             init=kk.KK_INIT_EMPTY if start is not None else kk.KK_INIT_RANDOM)
    if start is not None:
        L.set_lattice(start)
        ref = [start[r].copy() for r in range(R)]
    else:
        ref = [O.init_random(Lx, Ly, f, seed, replica=r) for r in range(R)]
    nab0 = L.energy()[0]
    L.sweep(n)
    got = L.get_lattice()
    st = L.stats()
    nab1 = L.energy()[0]
    for r in range(R):
        ost = O.run(ref[r], omega, seed, n, replica=r)
        assert np.array_equal(got[r], ref[r]), f"lattice mismatch replica {r}"
        assert list(st[r]) == _oracle_stats(ost)
        assert nab1[r] == O.n_ab(ref[r])
        assert nab1[r] - nab0[r] == st[r][3]
    assert (L.composition() == [int(x.sum()) for x in ref]).all()
    return L, ref


def test_config0_64x64_1000_sweeps():
    """BASELINE configs[0]: 64x64, 50:50, omega=0.5, 1000 sweeps, fixed seed."""
    _run_parity(64, 64, 0.5, 0.5, 20240601, 1000)


@pytest.mark.parametrize("T", [1, 2, 4, 8])
def test_iters_per_pass_all_equal_oracle(T):
    _run_parity(96, 40, 0.5, 0.6, 77, 12, T=T, env={"KK_RESIDENT": 0})   # tile kernel


@pytest.mark.parametrize("Lx,Ly,env", [
    (4, 4, None), (12, 8, None), (20, 12, None), (36, 40, {"KK_TWI": 1, "KK_THI": 8}),
    (8, 4, None), (16, 8, None), (40, 12, None), (72, 20, None),
    (200, 52, {"KK_TWI": 2, "KK_THI": 16}),      # many tiles, ragged last tile (W=7)
    (1000, 44, {"KK_TWI": 5, "KK_THI": 12}),     # Lx % 32 = 8, ragged in x and y
    (2048, 64, {"KK_TWI": 16, "KK_THI": 20}),
])
def test_sweep_parity_shapes(Lx, Ly, env):
    _run_parity(Lx, Ly, 0.5, 0.7, Lx * 31 + Ly, 6, env=env)


@pytest.mark.parametrize("omega", [0.0, 0.2, 1.0, -0.5, 4.0])
def test_sweep_parity_omega(omega):
    _run_parity(128, 32, 0.3, omega, 5, 10)


def test_replicas_and_arbitrary_start():
    start = inputs.random_lattice(64, 24, 0.45, seed=9, replicas=3)
    _run_parity(64, 24, 0.5, 0.8, 4242, 15, R=3, start=start)
    stripes = np.stack([inputs.striped_lattice(48, 16)] * 2)
    _run_parity(48, 16, 0.5, 1.0, 17, 20, R=2, start=stripes)


def test_degenerate_lattices():
    from paper_1309_4349_b200 import kk
    for f in (0.0, 1.0):
        L = _lat(32, 8, f, 0.5, 1)
        before = L.get_lattice()
        L.sweep(3)
        assert np.array_equal(L.get_lattice(), before)
        st = L.stats()[0]
        assert st[0] == 3 * 256 and st[1] == 3 * 256 and st[2] == 0
        assert L.energy()[0][0] == 0
        hist = L.cluster_histogram(1)[0]
        assert hist == ([(256, 1)] if f == 1.0 else [])
    L = _lat(32, 8, 0.5, 0.5, 1, init=kk.KK_INIT_EMPTY)
    L.sweep(0)
    assert L.sweep_index() == 0


@pytest.mark.parametrize("Lx,Ly,R", [(64, 64, 1), (400, 400, 2), (40, 12, 3)])
def test_cluster_histogram_parity(Lx, Ly, R):
    L, ref = _run_parity(Lx, Ly, 0.5, 0.9, 31, 20 if Lx < 400 else 5, R=R)
    for target in (0, 1):
        got = L.cluster_histogram(target)
        for r in range(R):
            assert got[r] == O.cluster_histogram(ref[r], target)


def test_cluster_histogram_large_clusters():
    """Sizes >= 4096 go through the big-cluster list: all-A, half-plane."""
    from paper_1309_4349_b200 import kk
    a = np.zeros((2, 128, 128), np.uint8)
    a[0] = 1
    a[1, :64] = 1
    a[1, 100, 5] = 1
    L = _lat(128, 128, 0.5, 0.5, 1, replicas=2, init=kk.KK_INIT_EMPTY)
    L.set_lattice(a)
    got = L.cluster_histogram(1)
    assert got[0] == [(128 * 128, 1)]
    assert got[1] == O.cluster_histogram(a[1], 1) == [(1, 1), (64 * 128, 1)]


def test_config1_400x400_paper_size():
    """BASELINE configs[1] shapes: 400x400 at 50:50 and 30:70 compositions."""
    for f, om in [(0.5, 0.6), (0.3, 1.0)]:
        L, ref = _run_parity(400, 400, f, om, 400, 3)   # resident kernel (default)
        assert L.cluster_histogram(1)[0] == O.cluster_histogram(ref[0], 1)


def test_config2_4096x4096_one_sweep():
    """BASELINE configs[2]: the single-B200 throughput lattice, full parity."""
    _run_parity(4096, 4096, 0.5, 0.6, 123, 1)


@pytest.mark.parametrize("T,init", [(4, "block"), (8, "random")])
def test_bench_lattice_65536_window_and_invariants(T, init):
    """BASELINE configs[4] lattice (65536 x 65536, what bench.py times; T = 8
    with the random start is bench.py's own launch configuration: the planar
    tile kernel with its cost-model tiles, TMA staging): invariants over the
    whole lattice + window parity for one full sweep (16 / T passes), with
    windows at tile seams (rows k * THI) and inside each TMA box of an
    interior band (the x seams lie inside every full-width window)."""
    from paper_1309_4349_b200 import kk
    Lx = Ly = 65536
    L = _lat(Lx, Ly, 0.5, 0.6, 99, init=kk.KK_INIT_BLOCK if init == "block" else kk.KK_INIT_RANDOM,
             iters_per_pass=T)
    pl = kk.plan(Lx, Ly, iters_per_pass=T)
    assert pl["kernel"] == "planar" and pl["tma_boxes"] >= 1
    nA = L.composition()[0]
    assert nA == Lx * Ly // 2
    L.sweep(1)                                    # mix the block start
    nab0 = L.energy()[0][0]
    L.stats(reset=True)
    passes = 16 // T
    hy = 3 * 16                                   # light cone of one sweep (R8)
    before = L.get_packed()[0]
    s = L.sweep_index()
    for _ in range(passes):                       # one sweep as single passes
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    after = L.get_packed()[0]
    st = L.stats()[0]
    nab1 = L.energy()[0][0]
    assert L.composition()[0] == nA
    assert nab1 - nab0 == st[3]
    assert st[0] == Lx * Ly                       # one sweep = N attempts (R11)
    THI, HYp = pl["tile_rows"], pl["halo_rows"]
    b = 5                                          # an interior band: staged rows b*THI - HYp ...
    box_rows = [b * THI - HYp + 8, b * THI - HYp + 250, b * THI - HYp + min(300, THI + 2 * HYp - 16)]
    seams = [0, THI - 4, 7 * THI - 4, Ly - 8]
    H = 8
    for y0 in seams + box_rows:
        rows = [(y0 - hy + r) % Ly for r in range(H + 2 * hy)]
        win = np.ascontiguousarray(inputs.unpack_rows(before[rows], Lx))
        O.window_iterations(win, Ly, y0 - hy, 0.6, 99, s, 0, 0, 16, hy, hy + H)
        exp = win[hy:hy + H]
        got = inputs.unpack_rows(after[[(y0 + r) % Ly for r in range(H)]], Lx)
        assert np.array_equal(got, exp), y0


def _forced_plan_parity(env, Lx, Ly, sweeps, kernel, boxes, monkeypatch, seed=777):
    """Full-lattice multi-sweep parity of a launch plan forced through the
    environment on a lattice the oracle finishes in seconds: 3 x 3 tiles, so
    the middle tile is staged by TMA (all its rows and groups inside the
    lattice) and the others exercise the x / y wrap through LDG."""
    from paper_1309_4349_b200 import kk
    for key, v in {**env, "KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 0, "KK_TMA": 1}.items():
        monkeypatch.setenv(key, str(v))
    p = kk.plan(Lx, Ly, n_sm=0)
    assert p["kernel"] == kernel and p["tiles_x"] == 3 and p["bands"] == 3, p
    assert p["tile_words"] == int(env["KK_TWI"]) and p["tile_rows"] == int(env["KK_THI"]), p
    assert p["tma_boxes"] == boxes, p
    if "KK_PASS_THREADS" in env:
        assert p["threads"] == int(env["KK_PASS_THREADS"])
    _run_parity(Lx, Ly, 0.5, 0.6, seed, sweeps)


def test_bench_plan_planar_full_parity(monkeypatch):
    """bench.py's 65536^2 plan (the planar kernel's cost-model tiles, CTA size,
    TMA boxes incl. the overlapped last box), forced on a 3 x 3-tile lattice."""
    from paper_1309_4349_b200 import kk
    pl = kk.plan(65536, 65536, n_sm=148)
    assert pl["kernel"] == "planar"
    env = {"KK_TWI": pl["tile_words"], "KK_THI": pl["tile_rows"], "KK_PASS_THREADS": pl["threads"],
           "KK_PDL": pl["pass_pdl"], "KK_PLANAR": 2}
    _forced_plan_parity(env, 3 * 32 * pl["tile_words"], 3 * pl["tile_rows"], 2, "planar", pl["tma_boxes"],
                        monkeypatch)


def test_bench_plan_planar_16384_full_parity(monkeypatch):
    from paper_1309_4349_b200 import kk
    pl = kk.plan(16384, 16384, n_sm=148)
    assert pl["kernel"] == "planar"
    env = {"KK_TWI": pl["tile_words"], "KK_THI": pl["tile_rows"], "KK_PASS_THREADS": pl["threads"],
           "KK_PDL": pl["pass_pdl"], "KK_PLANAR": 2}
    _forced_plan_parity(env, 3 * 32 * pl["tile_words"], 3 * pl["tile_rows"], 2, "planar", pl["tma_boxes"],
                        monkeypatch)


@pytest.mark.parametrize("twi,thi,nt,pdl,boxes", [(64, 596, 640, 0, 3), (64, 300, 512, 0, 2)])
def test_tile_kernel_tall_and_16384_plans_full_parity(twi, thi, nt, pdl, boxes, monkeypatch):
    """The row-major tile kernel's round-1 bench plan (64-word x 596-row tall
    tiles, 640 threads, 3 TMA boxes with an overlapped last box) and its
    16384^2 plan (300 rows, 512 threads, 2 boxes, PDL off), forced on 3 x 3
    tiles: the kernel every lattice with Lx % 128 != 0 (and every small one)
    runs."""
    env = {"KK_TWI": twi, "KK_THI": thi, "KK_PASS_THREADS": nt, "KK_PDL": pdl, "KK_PLANAR": 0}
    _forced_plan_parity(env, 3 * 32 * twi, 3 * thi, 2, "tile", boxes, monkeypatch)


def test_bench_lattice_65536_cluster_histogram():
    """The cluster histogram at the bench lattice size (65536 x 65536, the CCL
    launch configuration bench.py times), checked through a lattice whose
    clusters are known from a small oracle run: a random 256 x 256 tile with
    a B frame (row 0, column 0) inside an A ring (rows 1 and 255, columns 1
    and 255), repeated 256 x 256 times.  No A cluster and no interior B
    cluster can leave its tile (every neighbour step out of a tile lands on
    the frame or crosses it), so the big histogram is the tile's oracle
    histogram with every count x 65536, except that the frames of all tiles
    join into ONE B cluster of 511 x 65536 sites."""
    from paper_1309_4349_b200 import kk
    t, reps = 256, 256
    tile = inputs.random_lattice(t, t, 0.5, seed=4242)
    tile[1, :] = tile[t - 1, :] = 1
    tile[:, 1] = tile[:, t - 1] = 1
    tile[0, :] = 0
    tile[:, 0] = 0
    Lx = Ly = t * reps
    packed_tile = np.packbits(tile, axis=1, bitorder="little").view(np.uint32)  # bit x%32 of word x/32
    assert packed_tile.shape == (t, t // 32)
    big = np.tile(packed_tile, (reps, reps))[None]
    L = _lat(Lx, Ly, 0.5, 0.6, 1, init=kk.KK_INIT_EMPTY)
    L.set_packed(np.ascontiguousarray(big))
    del big
    assert np.array_equal(inputs.unpack_rows(L.get_packed()[0][:t, :t // 32], t), tile)
    n = reps * reps
    exp_a = [(sz, c * n) for sz, c in O.cluster_histogram(tile, 1)]
    hb = dict(O.cluster_histogram(tile, 0))
    hb[511] -= 1                                  # the frame on the tile torus
    exp_b = sorted([(sz, c * n) for sz, c in hb.items() if c] + [(511 * n, 1)])
    assert L.cluster_histogram(1)[0] == exp_a
    assert L.cluster_histogram(0)[0] == exp_b
    L.close()


def test_cluster_histogram_random_stress():
    """Random lattices over many shapes (several CCL tiles, ragged edges,
    replicas): the multiset must equal the oracle's every time (this caught a
    flatten-phase race in the tile kernel)."""
    from paper_1309_4349_b200 import kk
    rng = np.random.default_rng(11)
    for trial in range(40):
        Lx = int(rng.choice([8, 40, 256, 264, 400, 520, 1024]))
        Ly = int(rng.choice([4, 32, 36, 64, 100, 400]))
        R = int(rng.choice([1, 2, 3]))
        f = float(rng.choice([0.3, 0.5, 0.6, 0.7]))
        lat = inputs.random_lattice(Lx, Ly, f, seed=trial, replicas=R)
        L = _lat(Lx, Ly, 0.5, 0.5, 1, replicas=R, init=kk.KK_INIT_EMPTY)
        L.set_lattice(lat)
        for target in (0, 1):
            got = L.cluster_histogram(target)
            for r in range(R):
                assert got[r] == O.cluster_histogram(lat[r], target), (Lx, Ly, R, r, f, target)
        L.close()


@pytest.mark.parametrize("tma", [1, 0])
def test_tile_kernel_tma_staging_with_replicas(tma):
    """Interior tiles staged by TMA boxes (3D tensor map: word, row, replica)
    and edge tiles by LDG, with replicas, against the oracle; KK_TMA=0 forces
    LDG staging everywhere."""
    from paper_1309_4349_b200 import kk
    assert kk.plan(2048, 256, replicas=3)["kernel"] == "tile"
    _run_parity(2048, 256, 0.5, 0.7, 2048 + tma, 3, R=3, env={"KK_TMA": tma})


@pytest.mark.parametrize("pdl,Lx,Ly,env", [
    (1, 2048, 256, {}), (0, 2048, 256, {}),
    (1, 1000, 44, {"KK_TWI": 5, "KK_THI": 12}),    # Lx % 32 != 0: LDG staging, ragged tiles
])
def test_tile_kernel_programmatic_dependent_launch(pdl, Lx, Ly, env, monkeypatch):
    """Consecutive passes launched with programmatic stream serialization
    (the next pass's CTAs start before the previous pass ends and wait in
    griddepcontrol.wait before touching the lattice) against the oracle over
    several sweeps, forced on and off regardless of the grid size."""
    from paper_1309_4349_b200 import kk
    for key, v in {**env, "KK_PDL": pdl, "KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 0}.items():
        monkeypatch.setenv(key, str(v))
    p = kk.plan(Lx, Ly, replicas=2)
    assert p["kernel"] == "tile" and p["pass_pdl"] == pdl
    _run_parity(Lx, Ly, 0.5, 0.7, Lx + 17 * pdl, 4, R=2)


def test_tile_kernel_640_threads_default_5120(monkeypatch):
    """5120^2 is a one-wave grid of 180 x 32 tiles: the row-major tile kernel
    (KK_PLANAR=0) takes 640-thread CTAs (one per SM, up to 96 registers); one
    full sweep against the oracle."""
    from paper_1309_4349_b200 import kk
    monkeypatch.setenv("KK_PLANAR", "0")
    p = kk.plan(5120, 5120)
    assert p["kernel"] == "tile" and p["threads"] == 640
    _run_parity(5120, 5120, 0.5, 0.6, 5120, 1)


@pytest.mark.parametrize("Lx,Ly,env", [
    (2048, 256, {}),
    (1000, 44, {"KK_TWI": 5, "KK_THI": 12}),    # Lx % 32 != 0: per-centre draw path, LDG staging
])
def test_tile_kernel_640_threads_forced(Lx, Ly, env, monkeypatch):
    """KK_PASS_THREADS=640 on small and ragged shapes with replicas."""
    from paper_1309_4349_b200 import kk
    for key, v in {**env, "KK_PASS_THREADS": 640, "KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 0}.items():
        monkeypatch.setenv(key, str(v))
    p = kk.plan(Lx, Ly, replicas=2)
    assert p["kernel"] == "tile" and p["threads"] == 640
    _run_parity(Lx, Ly, 0.5, 0.7, Lx + 3, 3, R=2)


def test_cluster_histogram_total_over_replicas():
    """The replica-summed histogram equals the sum of the oracle's per-replica
    histograms (BASELINE configs[3]-style ensemble statistics)."""
    from collections import Counter
    L, ref = _run_parity(100, 40, 0.4, 0.9, 77, 6, R=5)
    for target in (0, 1):
        tot = Counter()
        for r in range(5):
            for sz, c in O.cluster_histogram(ref[r], target):
                tot[sz] += c
        assert L.cluster_histogram_total(target) == sorted(tot.items())


def test_8192_planar_default():
    """8192^2 runs on the planar tile kernel by default (it replaced the band
    kernel there); one full sweep must equal the oracle."""
    from paper_1309_4349_b200 import kk
    assert kk.plan(8192, 8192, n_sm=0)["kernel"] == "planar"
    _run_parity(8192, 8192, 0.5, 0.6, 8192, 1)


def test_12288_band_kernel_default_when_not_planar():
    """A lattice whose rows are not whole 128-site groups (Lx = 12000) takes
    the band kernel at this size; two sweeps against the oracle."""
    from paper_1309_4349_b200 import kk
    assert kk.plan(12000, 8192, n_sm=0)["kernel"] == "band"
    _run_parity(12000, 8192, 0.5, 0.6, 12000, 1)

"""Parity of the planar tile kernel (kk_planar.cu: plane-interleaved layout,
bit-sliced items, warp-compacted acceptance draws) with the oracle, through
the C ABI — bit-exact lattice, counters, N_AB, composition and cluster
histogram (north_star: "GPU results must match the oracle bit-exactly";
PAPER.md:150 "MPKK method generates the same results").

Covers: every T, forced small / ragged tiles (several tiles per row and per
column, last tile narrower), one tile spanning the whole row (x wrap inside
the tile), TMA on/off, PDL on/off, replicas, negative / zero / large omega
(draw side, no draws at all, draws that always fail), the block start,
mid-sweep starts through kk_pass, layout round trips between every call, and
seeded random configurations."""
import contextlib
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests import inputs
from tests.test_gpu_parity import _gpu  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


TILE_PATH = {"KK_RESIDENT": 0, "KK_CLUSTER": 0, "KK_BAND": 0, "KK_PLANAR": 2}


@contextlib.contextmanager
def _env(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update({k: str(v) for k, v in env.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _parity(Lx, Ly, f, omega, seed, n, T=0, env=None, R=1, start=None, split=0, ccl=True):
    from paper_1309_4349_b200 import kk
    with _env({**TILE_PATH, **(env or {})}):
        L = kk.Lattice(Lx, Ly, f, omega, seed, replicas=R, iters_per_pass=T,
                       init=kk.KK_INIT_EMPTY if start is not None else kk.KK_INIT_RANDOM)
        pl = kk.plan(Lx, Ly, replicas=R, iters_per_pass=T, n_sm=0)
    assert pl["kernel"] == "planar", pl
    if start is not None:
        L.set_lattice(start)
        ref = [start[r].copy() for r in range(R)]
    else:
        ref = [O.init_random(Lx, Ly, f, seed, replica=r) for r in range(R)]
    nab0 = L.energy()[0]
    Tp = pl["iters_per_pass"]
    for _ in range(split):                    # single passes (mid-sweep state), then whole sweeps
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
    L.sweep(n)
    done_iters = 16 * n + split * Tp
    full, rest = divmod(done_iters, 16)
    assert rest == 0, "tests keep whole sweeps"
    got = L.get_lattice()
    st = L.stats()
    nab1 = L.energy()[0]
    for r in range(R):
        ost = O.run(ref[r], omega, seed, full, replica=r)
        assert np.array_equal(got[r], ref[r]), f"lattice mismatch replica {r}"
        assert list(st[r]) == [ost["attempted"], ost["trivial"], ost["accepted"], ost["dnab_sum"]]
        assert nab1[r] == O.n_ab(ref[r])
        assert nab1[r] - nab0[r] == st[r][3]
    assert (L.composition() == [int(x.sum()) for x in ref]).all()
    if ccl:
        h = L.cluster_histogram(1)
        for r in range(R):
            assert h[r] == O.cluster_histogram(ref[r], 1)
    return L, ref


@pytest.mark.parametrize("T", [1, 2, 4, 8])
def test_planar_all_T(T):
    _parity(512, 256, 0.5, 0.6, 11 + T, 2, T=T)


@pytest.mark.parametrize("Lx,Ly,twi,thi", [(1024, 300, 16, 40), (640, 128, 32, 24), (384, 64, 8, 12),
                                           (128, 44, 4, 8), (896, 96, 64, 16)])
def test_planar_forced_tiles(Lx, Ly, twi, thi):
    """Several tiles per row (ragged last tile in x and y), one-group tiles,
    a tile as wide as the row (x halos wrap onto the same tile)."""
    _parity(Lx, Ly, 0.5, 0.7, Lx + Ly, 2, env={"KK_TWI": twi, "KK_THI": thi})


@pytest.mark.parametrize("tma,pdl", [(0, 0), (1, 1), (1, 0), (0, 1)])
def test_planar_tma_pdl(tma, pdl):
    _parity(2048, 512, 0.5, 0.6, 5, 2, env={"KK_TMA": tma, "KK_PDL": pdl, "KK_THI": 100})


@pytest.mark.parametrize("omega", [-0.7, 0.0, 3.0, 1e-12, -2.5])
def test_planar_omega_sides(omega):
    """omega < 0: draws for v < 0; omega = 0: no draw at all; large omega:
    draws that (nearly) always fail; tiny omega: thresholds of 2^32-1 on the
    draw side (drawn and accepted)."""
    _parity(768, 128, 0.4, omega, 77, 3)


def test_planar_replicas_and_block_start():
    from paper_1309_4349_b200 import kk
    _parity(256, 64, 0.3, 0.8, 3, 2, R=3)
    with _env(TILE_PATH):
        L = kk.Lattice(512, 128, 0.5, 0.6, 9, init=kk.KK_INIT_BLOCK)
    ref = O.init_block(512, 128, 0.5)
    L.sweep(3)
    O.run(ref, 0.6, 9, 3)
    assert np.array_equal(L.get_lattice()[0], ref)


def test_planar_split_passes_and_set_lattice():
    """kk_pass mid-sweep, then kk_sweep; an arbitrary start set through the ABI."""
    start = inputs.random_lattice(1024, 128, 0.45, seed=31)[None]
    _parity(1024, 128, 0.45, 0.9, 31, 1, T=4, split=4, start=start)
    stripes = inputs.striped_lattice(384, 96)[None]
    _parity(384, 96, 0.5, 0.5, 8, 2, T=8, split=2, start=stripes)


def test_planar_layout_round_trips():
    """Every public-layout call between passes converts back (get / energy /
    composition / clusters / packed copies) and the next pass converts again."""
    from paper_1309_4349_b200 import kk
    Lx, Ly, om, seed = 512, 64, 0.6, 4
    with _env(TILE_PATH):
        L = kk.Lattice(Lx, Ly, 0.5, om, seed, iters_per_pass=8)
    ref = O.init_random(Lx, Ly, 0.5, seed)
    for s in range(3):
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
        p = L.get_packed()                      # mid-sweep: layout restored
        L.set_packed(p.copy())                  # overwrite in the public layout
        L.run_pass(kk.REGION_ALL, None, None)
        L.pass_commit()
        O.run(ref, om, seed, 1, first_sweep=s)
        assert np.array_equal(L.get_lattice()[0], ref)
        assert L.energy()[0][0] == O.n_ab(ref)
        assert L.cluster_histogram(1)[0] == O.cluster_histogram(ref, 1)


def test_planar_long_run_1024():
    """20 sweeps of a 1024^2 lattice near the paper's microdomain regime."""
    _parity(1024, 1024, 0.5, 0.6, 1309, 20)


def _fuzz(n=24, seed=4349):
    rng = np.random.default_rng(seed)
    out = []
    for k in range(n):
        Lx = 128 * int(rng.integers(1, 9))
        Ly = 4 * int(rng.integers(2, 41))
        R = int(rng.choice([1, 1, 2]))
        T = int(rng.choice([1, 2, 4, 8]))
        omega = float(np.round(rng.uniform(-2.0, 3.0), 3))
        f = float(np.round(rng.uniform(0.0, 1.0), 3))
        twi = int(rng.choice([0, 4, 8, 16, 32]))
        thi = int(rng.choice([0, 8, 12, 20, 36]))
        out.append((k, Lx, Ly, R, T, omega, f, twi, thi))
    return out


@pytest.mark.parametrize("k,Lx,Ly,R,T,omega,f,twi,thi", _fuzz())
def test_planar_fuzz(k, Lx, Ly, R, T, omega, f, twi, thi):
    env = {}
    if twi:
        env["KK_TWI"] = twi
    if thi:
        env["KK_THI"] = thi
    _parity(Lx, Ly, f, omega, 7 * k + 1, 2, T=T, env=env, R=R, ccl=False)
